// The two W products of the AFN application (precond.py's Woodbury step restated for the AFN
// factor) for a point-major right-hand-side block (rows x k, a point's k values
// contiguous):
//   wy:  C (n2 x k) = alpha W Y + beta S,    W (n2 x m, row-major), Y (m x k)
//   wtu: Z (m x k)  = alpha W^T U + beta Y,  U (n2 x k)
// Both stream W (n2 * m * 8 bytes, 528 MB at configs[2]'s AFN) once and do 2 k flops per
// element: 8.25 flops per byte at k = 33, above the FP64 pipe's ridge (36 TF/s / 6.45 TB/s),
// so they are FP64-pipe bound. DMMA (mma.sync.m8n8k4.f64) does the contraction with the
// right-hand sides padded only to the next multiple of 8 (k = 33 -> 40 columns).
//
// W goes straight from HBM into the A fragments: the k index of every m8n8k4 step is
// permuted so a lane's two consecutive W elements (one 16-byte load) serve two k-steps (wy)
// or two m-tiles (wtu), and a warp's load covers whole 64/128-byte row segments. The small
// operand (Y: 270 KB; U: streamed once per j block) is read into the B fragments through
// L1/L2 with the same permutation. Every warp is independent (no shared memory, no barriers),
// so the work is split statically over exactly the resident warps: wy gives each warp a
// contiguous run of 8-row tiles (groups of up to 4, the last one masked), wtu gives each warp
// a 32-column block of Z and an equal share of the n2 rows, writing fixed-order partials that
// a finish pass adds in split order (deterministic).
#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {
namespace {

KGP_DEV void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

KGP_DEV double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

constexpr int WG_T = 128;  // threads per CTA (4 independent warps)
// m-tiles (8 rows / 8 columns of Z) per warp: 4, or 2 for wide blocks (register budget)
template <int NT>
struct Mt {
  static constexpr int V = NT <= 5 ? 4 : 2;
};
#ifndef WG_MINB
#define WG_MINB 2         // CTAs per SM the register budget is sized for (3: spills, slower)
#endif

struct WyArgs {
  int64_t n2, m, k;
  const double* w;  // (n2, m) row-major, row stride ldw
  int64_t ldw;
  const double* y;  // Y(j, c) = y[j * y_rs + c * y_cs]
  int64_t y_rs, y_cs;
  double* c;  // C(i, c) = c[i * c_rs + c * c_cs]
  int64_t c_rs, c_cs;
  const double* s;  // S, same shape, may be null
  int64_t s_rs, s_cs;
  double alpha, beta;
  int64_t nwarps;  // warps in the grid
};

// C = alpha W Y + beta S. Warp gw owns row groups [G gw / W, G (gw + 1) / W) of 8 WG_MT rows
// (G = ceil(n2 / (8 WG_MT))), one at a time (8 WG_MT rows x 8 NT columns of accumulators).
// Unit column strides (point-major Y, C, S). The main loop runs over the full 8-wide steps
// of j without predicates: rows past n2 read row n2 - 1 and columns past k read column k - 1
// (both only feed accumulators that are never stored); a masked step handles m % 8.
template <int NT>
__global__ void __launch_bounds__(WG_T, WG_MINB) wy_kernel(const WyArgs g) {
  constexpr int WG_MT = Mt<NT>::V;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * (WG_T / 32) + (threadIdx.x >> 5);
  const int64_t groups = (g.n2 + 8 * WG_MT - 1) / (8 * WG_MT);
  const int64_t t_beg = WG_MT * (groups * gw / g.nwarps), t_end = WG_MT * (groups * (gw + 1) / g.nwarps);
  const int64_t m = g.m, nfull = m / 8, yrs = g.y_rs;
  const int64_t clast = 8 * (NT - 1) + r < g.k ? 8 * (NT - 1) + r : g.k - 1;
  for (int64_t t0 = t_beg; t0 < t_end; t0 += WG_MT) {
    const double* wr[WG_MT];
#pragma unroll
    for (int t = 0; t < WG_MT; ++t) {
      const int64_t i = 8 * (t0 + t) + r;
      wr[t] = g.w + (i < g.n2 ? i : g.n2 - 1) * g.ldw + 2 * q;
    }
    // B (k-step h, n-tile u) = Y[8 s + 2 q + h][8 u + r]: rows 2q (+1) of the step
    const double* yb = g.y + 2 * q * yrs + r;
    const double* yl = g.y + 2 * q * yrs + clast;
    double acc[WG_MT][NT][2];
#pragma unroll
    for (int t = 0; t < WG_MT; ++t)
#pragma unroll
      for (int u = 0; u < NT; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
    auto load_a = [&](int64_t s, double2(&a)[WG_MT]) {
#pragma unroll
      for (int t = 0; t < WG_MT; ++t) a[t] = ldg2(wr[t] + 8 * s);
    };
    auto load_b = [&](int64_t s, double2(&b)[NT]) {
      const double* p = yb + 8 * s * yrs;
      const double* pl = yl + 8 * s * yrs;
#pragma unroll
      for (int u = 0; u < NT - 1; ++u) b[u] = make_double2(__ldg(p + 8 * u), __ldg(p + yrs + 8 * u));
      b[NT - 1] = make_double2(__ldg(pl), __ldg(pl + yrs));
    };
    auto mma_step = [&](const double2(&a)[WG_MT], const double2(&b)[NT]) {
      // the two k-steps in separate sweeps: a DMMA's accumulator was last written 4 NT
      // (independent) DMMAs earlier
#pragma unroll
      for (int t = 0; t < WG_MT; ++t)
#pragma unroll
        for (int u = 0; u < NT; ++u) dmma(acc[t][u], a[t].x, b[u].x);
#pragma unroll
      for (int t = 0; t < WG_MT; ++t)
#pragma unroll
        for (int u = 0; u < NT; ++u) dmma(acc[t][u], a[t].y, b[u].y);
    };
    if (nfull > 0) {
      double2 a0[WG_MT], a1[WG_MT], b0[NT], b1[NT];
      load_a(0, a0);
      if (nfull > 1) load_a(1, a1);
      load_b(0, b0);
      for (int64_t s = 0; s < nfull; s += 2) {
        if (s + 1 < nfull) load_b(s + 1, b1);
        mma_step(a0, b0);
        if (s + 2 < nfull) load_a(s + 2, a0);
        if (s + 1 < nfull) {
          if (s + 2 < nfull) load_b(s + 2, b0);
          mma_step(a1, b1);
          if (s + 3 < nfull) load_a(s + 3, a1);
        }
      }
    }
    if (m % 8) {  // masked last step (m even: a lane's pair is valid or not as a whole)
      const bool jv = 8 * nfull + 2 * q < m;
      double2 a[WG_MT], b[NT];
#pragma unroll
      for (int t = 0; t < WG_MT; ++t) a[t] = jv ? ldg2(wr[t] + 8 * nfull) : make_double2(0.0, 0.0);
      if (jv) {
        load_b(nfull, b);
      } else {
#pragma unroll
        for (int u = 0; u < NT; ++u) b[u] = make_double2(0.0, 0.0);
      }
      mma_step(a, b);
    }
#pragma unroll
    for (int t = 0; t < WG_MT; ++t) {
      const int64_t i = 8 * (t0 + t) + r;
      if (i >= g.n2) continue;
#pragma unroll
      for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t c = 8 * u + 2 * q + h;
          if (c >= g.k) continue;
          double v = g.alpha * acc[t][u][h];
          if (g.s) v += g.beta * g.s[i * g.s_rs + c];
          g.c[i * g.c_rs + c] = v;
        }
    }
  }
}

struct WtuArgs {
  int64_t n2, m, k;
  const double* w;
  int64_t ldw;
  const double* u;  // U(i, c) = u[i * u_rs + c], unit column stride
  int64_t u_rs;
  double* part;  // part[split][j][c], (m x k) row-major per split
  int64_t jblocks, nsplit;
};

// part[split] = W[rows of split, :]^T U[rows of split, :]. Warp gw: column block gw % jblocks
// (8 WG_MT output rows j x 8 NT columns), row split gw / jblocks. Main loop over full 8-row
// steps without predicates (columns past m / k read valid neighbours that only feed
// accumulators never stored); a masked step handles the split's last rows.
template <int NT>
__global__ void __launch_bounds__(WG_T, WG_MINB) wtu_kernel(const WtuArgs g) {
  constexpr int WG_MT = Mt<NT>::V;
  const int lane = threadIdx.x & 31;
  const int a8 = lane >> 2, q = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * (WG_T / 32) + (threadIdx.x >> 5);
  if (gw >= g.jblocks * g.nsplit) return;
  const int64_t jb = (gw % g.jblocks) * (WG_MT * 8), split = gw / g.jblocks;
  const int64_t steps_all = (g.n2 + 7) / 8;
  const int64_t i_beg = 8 * (steps_all * split / g.nsplit);
  const int64_t i_end_raw = 8 * (steps_all * (split + 1) / g.nsplit);
  const int64_t i_end = i_end_raw < g.n2 ? i_end_raw : g.n2;
  const int64_t m = g.m, ldw = g.ldw, urs = g.u_rs;
  double acc[WG_MT][NT][2];
#pragma unroll
  for (int t = 0; t < WG_MT; ++t)
#pragma unroll
    for (int u = 0; u < NT; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  // A (k-step h, m-tile pair p) = W[i_beg + 8 s + 2 q + h][jb + 16 p + 2 a8 (+1)], the column
  // clamped to the last pair (m even)
  const double* wa[WG_MT / 2];
#pragma unroll
  for (int p = 0; p < WG_MT / 2; ++p) {
    const int64_t j = jb + 16 * p + 2 * a8;
    wa[p] = g.w + (i_beg + 2 * q) * ldw + (j < m ? j : m - 2);
  }
  // B (k-step h, n-tile u) = U[i_beg + 8 s + 2 q + h][8 u + a8], the last tile's column clamped
  const int64_t clast = 8 * (NT - 1) + a8 < g.k ? 8 * (NT - 1) + a8 : g.k - 1;
  const double* ub = g.u + (i_beg + 2 * q) * urs + a8;
  const double* ul = g.u + (i_beg + 2 * q) * urs + clast;
  auto load_a = [&](int64_t s, double2(&a)[WG_MT / 2][2]) {
#pragma unroll
    for (int p = 0; p < WG_MT / 2; ++p) {
      a[p][0] = ldg2(wa[p] + 8 * s * ldw);
      a[p][1] = ldg2(wa[p] + (8 * s + 1) * ldw);
    }
  };
  auto load_b = [&](int64_t s, double2(&b)[NT]) {
    const double* p = ub + 8 * s * urs;
    const double* pl = ul + 8 * s * urs;
#pragma unroll
    for (int u = 0; u < NT - 1; ++u) b[u] = make_double2(__ldg(p + 8 * u), __ldg(p + urs + 8 * u));
    b[NT - 1] = make_double2(__ldg(pl), __ldg(pl + urs));
  };
  auto mma_step = [&](const double2(&a)[WG_MT / 2][2], const double2(&b)[NT]) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int p = 0; p < WG_MT / 2; ++p)
#pragma unroll
        for (int u = 0; u < NT; ++u) {
          const double bv = h ? b[u].y : b[u].x;
          dmma(acc[2 * p][u], h ? a[p][1].x : a[p][0].x, bv);
          dmma(acc[2 * p + 1][u], h ? a[p][1].y : a[p][0].y, bv);
        }
  };
  const int64_t nfull = (i_end - i_beg) / 8;
  if (nfull > 0) {
    double2 a0[WG_MT / 2][2], a1[WG_MT / 2][2], b0[NT], b1[NT];
    load_a(0, a0);
    if (nfull > 1) load_a(1, a1);
    load_b(0, b0);
    for (int64_t s = 0; s < nfull; s += 2) {
      if (s + 1 < nfull) load_b(s + 1, b1);
      mma_step(a0, b0);
      if (s + 2 < nfull) load_a(s + 2, a0);
      if (s + 1 < nfull) {
        if (s + 2 < nfull) load_b(s + 2, b0);
        mma_step(a1, b1);
        if (s + 3 < nfull) load_a(s + 3, a1);
      }
    }
  }
  if ((i_end - i_beg) % 8) {  // masked last step: rows past the split contribute zero
    const int64_t i0 = i_beg + 8 * nfull + 2 * q;
    const bool v0 = i0 < i_end, v1 = i0 + 1 < i_end;
    double2 a[WG_MT / 2][2], b[NT];
#pragma unroll
    for (int p = 0; p < WG_MT / 2; ++p) {
      a[p][0] = v0 ? ldg2(wa[p] + 8 * nfull * ldw) : make_double2(0.0, 0.0);
      a[p][1] = v1 ? ldg2(wa[p] + (8 * nfull + 1) * ldw) : make_double2(0.0, 0.0);
    }
    const double* p = ub + 8 * nfull * urs;
    const double* pl = ul + 8 * nfull * urs;
#pragma unroll
    for (int u = 0; u < NT - 1; ++u)
      b[u] = make_double2(v0 ? __ldg(p + 8 * u) : 0.0, v1 ? __ldg(p + urs + 8 * u) : 0.0);
    b[NT - 1] = make_double2(v0 ? __ldg(pl) : 0.0, v1 ? __ldg(pl + urs) : 0.0);
    mma_step(a, b);
  }
  // C fragment: row a8 of m-tile 2p + e is j = jb + 16 p + 2 a8 + e; columns 8 u + 2 q + h
  double* out = g.part + split * m * g.k;
#pragma unroll
  for (int p = 0; p < WG_MT / 2; ++p)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t j = jb + 16 * p + 2 * a8 + e;
      if (j >= m) continue;
#pragma unroll
      for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t c = 8 * u + 2 * q + h;
          if (c < g.k) out[j * g.k + c] = acc[2 * p + e][u][h];
        }
    }
}

// z[j, c] = alpha * sum_s part[s][j][c] + beta * src[j, c], fixed order in s
__global__ void wtu_finish_kernel(int64_t m, int64_t k, int ns, const double* __restrict__ part, double alpha,
                                  double beta, const double* __restrict__ src, int64_t s_rs, int64_t s_cs,
                                  double* __restrict__ z, int64_t z_rs, int64_t z_cs) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * k) return;
  const int64_t j = e / k, c = e - j * k;
  double acc = 0.0;
  for (int s = 0; s < ns; ++s) acc += part[(int64_t)s * m * k + e];
  double v = alpha * acc;
  if (src) v += beta * src[j * s_rs + c * s_cs];
  z[j * z_rs + c * z_cs] = v;
}

// resident warps of kernel f on the current device (occupancy x SMs x 4)
template <typename K>
int64_t resident_warps(K f) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, WG_T, 0);
  if (sms <= 0) sms = 148;
  if (per_sm <= 0) per_sm = 1;
  return (int64_t)sms * per_sm * (WG_T / 32);
}

template <int NT>
int wy_launch(WyArgs g, cudaStream_t st) {
  constexpr int WG_MT = Mt<NT>::V;
  // every warp the same number of row groups (the smallest warp count that keeps the
  // per-warp maximum of a resident-warp split)
  const int64_t groups = (g.n2 + 8 * WG_MT - 1) / (8 * WG_MT);
  const int64_t res = resident_warps(wy_kernel<NT>);
  const int64_t per = (groups + res - 1) / res;
  int64_t nw = (groups + per - 1) / per;
  if (nw < 1) nw = 1;
  nw = (nw + 3) / 4 * 4;
  g.nwarps = nw;
  wy_kernel<NT><<<(unsigned)(nw / 4), WG_T, 0, st>>>(g);
  KGP_LAUNCH("wy_kernel");
  return KGP_OK;
}

template <int NT>
int wtu_launch(WtuArgs g, double alpha, double beta, const double* src, int64_t s_rs, int64_t s_cs, double* z,
               int64_t z_rs, int64_t z_cs, DevBuf& tmp, cudaStream_t st) {
  constexpr int WG_MT = Mt<NT>::V;
  const int64_t nw = resident_warps(wtu_kernel<NT>);
  g.jblocks = (g.m + WG_MT * 8 - 1) / (WG_MT * 8);
  int64_t ns = nw / g.jblocks;
  const int64_t max_ns = (g.n2 + 127) / 128;  // >= 128 rows per split
  if (ns > max_ns) ns = max_ns;
  if (ns < 1) ns = 1;
  g.nsplit = ns;
  int rc = tmp.ensure(sizeof(double) * (size_t)(ns * g.m * g.k));
  if (rc) return rc;
  g.part = tmp.as<double>();
  const int64_t warps = g.jblocks * ns;
  wtu_kernel<NT><<<(unsigned)((warps + 3) / 4), WG_T, 0, st>>>(g);
  KGP_LAUNCH("wtu_kernel");
  wtu_finish_kernel<<<(unsigned)((g.m * g.k + 255) / 256), 256, 0, st>>>(g.m, g.k, (int)ns, g.part, alpha, beta,
                                                                         src, s_rs, s_cs, z, z_rs, z_cs);
  KGP_LAUNCH("wtu_finish_kernel");
  return KGP_OK;
}

}  // namespace

bool wgemm_supported(int64_t m, int64_t k, const double* w, int64_t ldw) {
  return k >= 1 && k <= 64 && m >= 2 && (int64_t)k * 8 < INT32_MAX && (m % 2) == 0 && (ldw % 2) == 0 && (((uintptr_t)w) & 15) == 0;
}

int wy_product(int64_t n2, int64_t m, int64_t k, const double* w, int64_t ldw, const double* y, int64_t y_rs,
               int64_t y_cs, double* c, int64_t c_rs, int64_t c_cs, double alpha, double beta, const double* s,
               int64_t s_rs, int64_t s_cs, cudaStream_t st) {
  if (n2 <= 0 || k <= 0) return KGP_OK;
  KGP_REQUIRE(y_cs == 1 && c_cs == 1 && (s == nullptr || s_cs == 1), KGP_ERR_INVALID,
              "wy_product: unit column strides required");
  const WyArgs g{n2, m, k, w, ldw, y, y_rs, y_cs, c, c_rs, c_cs, s, s_rs, s_cs, alpha, beta, 0};
  switch ((k + 7) / 8) {
#define KGP_WY(NT) \
  case NT: return wy_launch<NT>(g, st);
    KGP_WY(1) KGP_WY(2) KGP_WY(3) KGP_WY(4) KGP_WY(5) KGP_WY(6) KGP_WY(7) KGP_WY(8)
#undef KGP_WY
  }
  KGP_REQUIRE(false, KGP_ERR_INVALID, "wy_product: k = %lld > 64", (long long)k);
}

int wtu_product(int64_t n2, int64_t m, int64_t k, const double* w, int64_t ldw, const double* u, int64_t u_rs,
                int64_t u_cs, double* z, int64_t z_rs, int64_t z_cs, double alpha, double beta, const double* src,
                int64_t s_rs, int64_t s_cs, DevBuf& tmp, cudaStream_t st) {
  if (m <= 0 || k <= 0) return KGP_OK;
  KGP_REQUIRE(u_cs == 1, KGP_ERR_INVALID, "wtu_product: unit column stride required");
  const WtuArgs g{n2, m, k, w, ldw, u, u_rs, nullptr, 0, 0};
  switch ((k + 7) / 8) {
#define KGP_WT(NT) \
  case NT: return wtu_launch<NT>(g, alpha, beta, src, s_rs, s_cs, z, z_rs, z_cs, tmp, st);
    KGP_WT(1) KGP_WT(2) KGP_WT(3) KGP_WT(4) KGP_WT(5) KGP_WT(6) KGP_WT(7) KGP_WT(8)
#undef KGP_WT
  }
  KGP_REQUIRE(false, KGP_ERR_INVALID, "wtu_product: k = %lld > 64", (long long)k);
}

}  // namespace kgp
