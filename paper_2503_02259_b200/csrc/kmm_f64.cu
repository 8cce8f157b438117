// Fused kernel-matrix MatMul in fp64 (precision KGP_FP64): the parity anchor.
//
// Same contract as KernelEngine._streamed_matmul (kmat.py:165-189): per entry a
// direct-difference r^2 in fp64 (_panels_numba.py:23-34 order, no FMA
// contraction), the kernel and its l-derivative (_panels_numba.py:37-131),
// contracted against the RHS block in fp64. Khat is never stored, not even a tile:
//
// one thread = one row. A CTA of 128 threads stages a tile of TJ column points and the
// matching RHS rows in shared memory; every thread evaluates kappa (and dkappa/dl) of its
// row against each column and FMAs it straight into its KS register accumulators (the
// column data are warp-broadcast reads). The RHS is processed in slices of KS <= 24/32
// columns (grid.y); when the row blocks cannot fill the GPU the column range is split
// over grid.z and the partial sums are reduced in a fixed order (deterministic).
// Bound: the FP64 pipe (distance 3d + exp ~25 + KS FMA per entry and output).
#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

constexpr int NT = 128;  // threads = rows per CTA
constexpr int TJ = 64;   // columns per shared-memory tile
constexpr int MAXD = 16;

template <int KT, int NOUT, int KS, int DB>
__global__ void __launch_bounds__(NT) kmm_f64_kernel(const F64Params p) {
  if (p.gate != nullptr && *p.gate == 0) return;  // PCG iteration past convergence
  __shared__ double sXj[TJ][DB + 1];
  __shared__ __align__(16) double sB[TJ][KS];

  const int tid = threadIdx.x;
  const int64_t r = (int64_t)blockIdx.x * NT + tid;
  const int c0 = blockIdx.y * KS;  // RHS slice
  const int d = p.d;
  const int64_t jb = (int64_t)blockIdx.z * p.jchunk;
  const int64_t je = jb + p.jchunk < p.ncols ? jb + p.jchunk : p.ncols;
  const bool live = r < p.nrows;

  double xi[DB];  // DB: d rounded up to 4, 8 or 16 (register budget)
#pragma unroll
  for (int q = 0; q < DB; ++q) xi[q] = (live && q < d) ? p.xr[r * d + q] : 0.0;
  double acc[KS], accg[NOUT == 2 ? KS : 1];
#pragma unroll
  for (int c = 0; c < KS; ++c) {
    acc[c] = 0.0;
    if (NOUT == 2) accg[c] = 0.0;
  }

  for (int64_t j0 = jb; j0 < je; j0 += TJ) {
    const int nj = (int)(je - j0 < TJ ? je - j0 : TJ);
    __syncthreads();
    for (int e = tid; e < nj * d; e += NT) sXj[e / d][e % d] = p.xc[(j0 + e / d) * d + e % d];
    for (int e = tid; e < nj * KS; e += NT) {
      const int jj = e / KS, c = e % KS;
      const int cc = c0 + c;
      sB[jj][c] = cc < p.k ? p.b[(j0 + jj) * p.b_rs + (int64_t)cc * p.b_cs] : 0.0;
    }
    __syncthreads();
    for (int jj = 0; jj < nj; ++jj) {
      double r2 = 0.0;
#pragma unroll
      for (int q = 0; q < DB; ++q) {
        if (q < d) {
          const double df = xi[q] - sXj[jj][q];
          r2 = __dadd_rn(r2, __dmul_rn(df, df));  // numba's rounding (no FMA contraction)
        }
      }
      const double kv = kappa64<KT>(r2, p.l);
      const double gv = NOUT == 2 ? dkappa64<KT>(r2, p.l) : 0.0;
#pragma unroll
      for (int c = 0; c < KS; c += 2) {
        const double2 bv = *reinterpret_cast<const double2*>(&sB[jj][c]);
        acc[c] = fma(kv, bv.x, acc[c]);
        acc[c + 1] = fma(kv, bv.y, acc[c + 1]);
        if (NOUT == 2) {
          accg[c] = fma(gv, bv.x, accg[c]);
          accg[c + 1] = fma(gv, bv.y, accg[c + 1]);
        }
      }
    }
  }
  if (!live) return;
  // epilogue (kmat.py:186-188): scale, + s B on the diagonal rows; raw partials when split
#pragma unroll
  for (int c = 0; c < KS; ++c) {
    const int cc = c0 + c;
    if (cc >= p.k) continue;
    if (p.part) {
      const int64_t slot = ((int64_t)blockIdx.z * p.nrows + r) * p.k + cc;
      p.part[slot] = acc[c];
      if (NOUT == 2) p.part[p.part_stride + slot] = accg[c];
      continue;
    }
    const int64_t o = r * p.o_rs + (int64_t)cc * p.o_cs;
    if (p.out_k) {
      double v = p.f2 * acc[c];
      if (p.diag_row0 >= 0) v += p.s * p.b[(p.diag_row0 + r) * p.b_rs + (int64_t)cc * p.b_cs];
      p.out_k[o] = v;
    }
    if (p.out_df) p.out_df[o] = p.two_f * acc[c];
    if (NOUT == 2 && p.out_dl) p.out_dl[o] = p.f2_dl * accg[c];
  }
}

// sum the column-split partials in split order, then the epilogue
__global__ void f64_reduce_kernel(const F64Params p, int nsplit) {
  if (p.gate != nullptr && *p.gate == 0) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.nrows * p.k) return;
  const int64_t r = e / p.k;
  const int c = (int)(e % p.k);
  double a = 0.0, g = 0.0;
  for (int z = 0; z < nsplit; ++z) {
    a += p.part[(int64_t)z * p.nrows * p.k + e];
    if (p.out_dl) g += p.part[p.part_stride + (int64_t)z * p.nrows * p.k + e];
  }
  const int64_t o = r * p.o_rs + (int64_t)c * p.o_cs;
  if (p.out_k) {
    double v = p.f2 * a;
    if (p.diag_row0 >= 0) v += p.s * p.b[(p.diag_row0 + r) * p.b_rs + (int64_t)c * p.b_cs];
    p.out_k[o] = v;
  }
  if (p.out_df) p.out_df[o] = p.two_f * a;
  if (p.out_dl) p.out_dl[o] = p.f2_dl * g;
}

// RHS slice width: the fewest slices within the register budget (24 columns with two
// outputs, 48 with one), each rounded up to a multiple of 4 -- every slice re-evaluates
// the kernel entries, so k = 33 runs as one slice of 36, not 32 + 4
inline int slice_for(int k, int nout) {
  const int cap = nout == 2 ? 24 : 48;
  const int nsl = (k + cap - 1) / cap;
  return ((k + nsl - 1) / nsl + 3) / 4 * 4;
}

template <int KT, int NOUT, int DB>
int launch_ks(const F64Params& p, int ks, dim3 grid, cudaStream_t st) {
  switch (ks) {
#define KGP_F64_KS(K)                                                      \
  case K:                                                                  \
    if constexpr (NOUT == 1 || K <= 24) {                                  \
      kmm_f64_kernel<KT, NOUT, K, DB><<<grid, NT, 0, st>>>(p);             \
      break;                                                               \
    }                                                                      \
    [[fallthrough]];
    KGP_F64_KS(4) KGP_F64_KS(8) KGP_F64_KS(12) KGP_F64_KS(16) KGP_F64_KS(20) KGP_F64_KS(24) KGP_F64_KS(28)
    KGP_F64_KS(32) KGP_F64_KS(36) KGP_F64_KS(40) KGP_F64_KS(44) KGP_F64_KS(48)
#undef KGP_F64_KS
    default:
      set_error(KGP_ERR_INVALID, "fp64 operator slice %d unsupported", ks);
      return KGP_ERR_INVALID;
  }
  KGP_LAUNCH("kmm_f64_kernel");
  return KGP_OK;
}

template <int KT>
int launch_kt(const F64Params& p, int ks, dim3 grid, cudaStream_t st) {
  const bool two = p.out_dl != nullptr;
  if (p.d <= 4) return two ? launch_ks<KT, 2, 4>(p, ks, grid, st) : launch_ks<KT, 1, 4>(p, ks, grid, st);
  if (p.d <= 8) return two ? launch_ks<KT, 2, 8>(p, ks, grid, st) : launch_ks<KT, 1, 8>(p, ks, grid, st);
  return two ? launch_ks<KT, 2, 16>(p, ks, grid, st) : launch_ks<KT, 1, 16>(p, ks, grid, st);
}

}  // namespace

int launch_kmm_f64(int kt, const F64Params& p_in, DevBuf& ws, cudaStream_t st) {
  KGP_REQUIRE(p_in.d >= 1 && p_in.d <= MAXD, KGP_ERR_INVALID, "fp64 operator supports 1 <= d <= %d, got %d", MAXD,
              p_in.d);
  KGP_REQUIRE(kt >= 0 && kt <= 2, KGP_ERR_INVALID, "unknown kernel id %d", kt);
  if (p_in.nrows <= 0) return KGP_OK;
  F64Params p = p_in;
  const int nout = p.out_dl ? 2 : 1;
  const int ks = slice_for(p.k, nout);
  const int64_t rblk = (p.nrows + NT - 1) / NT, kslc = (p.k + ks - 1) / ks;
  // split the columns until ~8 CTAs per SM are in flight (148 SMs), at >= 128 columns per split
  int64_t nsplit = (8 * 148 + rblk * kslc - 1) / (rblk * kslc);
  const int64_t maxsplit = p.ncols / 128 > 0 ? p.ncols / 128 : 1;
  if (nsplit > maxsplit) nsplit = maxsplit;
  if (nsplit > 65535) nsplit = 65535;
  if (nsplit < 1) nsplit = 1;
  p.jchunk = ((p.ncols + nsplit - 1) / nsplit + TJ - 1) / TJ * TJ;
  nsplit = (p.ncols + p.jchunk - 1) / p.jchunk;
  p.part = nullptr;
  p.part_stride = 0;
  if (nsplit > 1) {
    const int64_t per = nsplit * p.nrows * p.k;
    int rc = ws.ensure(sizeof(double) * per * (p.out_dl ? 2 : 1));
    if (rc) return rc;
    p.part = ws.as<double>();
    p.part_stride = per;
  }
  dim3 grid((unsigned)rblk, (unsigned)kslc, (unsigned)nsplit);
  int rc = (kt == GAUSS) ? launch_kt<GAUSS>(p, ks, grid, st) : (kt == MAT32) ? launch_kt<MAT32>(p, ks, grid, st)
                                                                                : launch_kt<MAT52>(p, ks, grid, st);
  if (rc || nsplit == 1) return rc;
  const int64_t cnt = p.nrows * p.k;
  f64_reduce_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(p, (int)nsplit);
  KGP_LAUNCH("f64_reduce_kernel");
  return KGP_OK;
}

}  // namespace kgp
