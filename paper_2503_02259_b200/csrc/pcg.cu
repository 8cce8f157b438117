// Device-resident batched PCG, SLQ log-determinant and NLML+gradient assembly.
//
// pcg_solve (solver.py:122-192): the k right-hand sides share one fused
// operator call per iteration (frozen columns included, solver.py:158); the
// per-column alpha/beta recurrences, breakdown checks and the freeze decision
// run in small device kernels, and the host reads back one status word per
// iteration. State is (k, n): column c contiguous (the reference's transposed
// layout, solver.py:143-146), which makes every per-column dot a contiguous
// reduction and every operator output write coalesced.
//
// slq_logdet (solver.py:238-265): one thread per probe rebuilds the Lanczos
// tridiagonal from the CG coefficients (solver.py:220-235) and diagonalises it
// with implicit-shift QL, tracking only the first row of the eigenvector
// matrix (all that e1^T log(T) e1 needs).
//
// nlml_grad_iterative (gp.py:133-179): PCG w-solve, unpreconditioned probe
// solves, SLQ, then one fused derivative pass over V = [w, Z] producing
// dKhat/dl V and dKhat/df V together.
#include <math.h>
#include <string.h>

#include <vector>

#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

constexpr int DOT_THREADS = 256;
constexpr int DOT_CHUNK = 8192;  // elements per block in the first reduction pass
constexpr int HIST = 4;          // ints per iteration in the mapped history

// elements per block of dot_fused_kernel (env KGP_DOT_CHUNK overrides)
int fused_chunk() {
  static const int v = [] {
    const char* s = getenv("KGP_DOT_CHUNK");
    const int c = s ? atoi(s) : DOT_CHUNK;
    return c < 256 ? 256 : c;
  }();
  return v;
}

// partial[c * nb + blk] = sum over the block's chunk of a[c*n+i] * b[c*n+i]
__global__ void dot_partial_kernel(int64_t n, int nb, const double* __restrict__ a, const double* __restrict__ b,
                                   double* __restrict__ partial) {
  const int c = blockIdx.y, blk = blockIdx.x;
  const double* ac = a + (int64_t)c * n;
  const double* bc = b + (int64_t)c * n;
  const int64_t i0 = (int64_t)blk * DOT_CHUNK;
  const int64_t i1 = i0 + DOT_CHUNK < n ? i0 + DOT_CHUNK : n;
  double s = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += DOT_THREADS) s = fma(ac[i], bc[i], s);
  __shared__ double red[DOT_THREADS / 32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < DOT_THREADS / 32 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) partial[(int64_t)c * nb + blk] = v;
  }
}

__global__ void dot_final_kernel(int k, int nb, const double* __restrict__ partial, double* __restrict__ out) {
  const int c = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += 32) s += partial[(int64_t)c * nb + i];
  s = warp_sum(s);
  if (threadIdx.x == 0) out[c] = s;
}

// One-launch column dots for the PCG loop: out[c] = a_c . b_c (c < k) and, when a2 is
// given, out2[c] = a2_c . b2_c (c < k2). Each block writes its chunk's partials; the last
// block of a column (ticket counter) sums them in block order -- the same fixed order as
// dot_partial + dot_final, so results are run-to-run identical -- and re-arms the ticket.
// Block sums of a[i] b[i] (and a2[i] b2[i] when two) over [i0, i1) of one column (offset
// off); the totals are valid in warp 0. Four independent accumulators per thread: four
// loads in flight (the loop is latency-bound for the short columns of small problems),
// combined in a fixed order. Every thread of the block must call it.
template <int DT>
KGP_DEV void block_dots(int64_t off, int64_t i0, int64_t i1, const double* __restrict__ a,
                        const double* __restrict__ b, const double* __restrict__ a2, const double* __restrict__ b2,
                        bool two, double& v, double& v2) {
  double sa[4] = {0.0, 0.0, 0.0, 0.0}, sb[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t i = i0 + threadIdx.x;
  for (; i + 3 * DT < i1; i += 4 * DT) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = off + i + u * DT;
      sa[u] = fma(a[j], b[j], sa[u]);
      if (two) sb[u] = fma(a2[j], b2[j], sb[u]);
    }
  }
  for (; i < i1; i += DT) {
    sa[0] = fma(a[off + i], b[off + i], sa[0]);
    if (two) sb[0] = fma(a2[off + i], b2[off + i], sb[0]);
  }
  double s = (sa[0] + sa[1]) + (sa[2] + sa[3]);
  double s2 = (sb[0] + sb[1]) + (sb[2] + sb[3]);
  __shared__ double red[2][DT / 32];
  s = warp_sum(s);
  s2 = warp_sum(s2);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s;
    red[1][threadIdx.x >> 5] = s2;
  }
  __syncthreads();
  v = v2 = 0.0;
  if (threadIdx.x < 32) {
    v = threadIdx.x < DT / 32 ? red[0][threadIdx.x] : 0.0;
    v2 = threadIdx.x < DT / 32 ? red[1][threadIdx.x] : 0.0;
    v = warp_sum(v);
    v2 = warp_sum(v2);
  }
}

template <int DT>
__global__ void __launch_bounds__(DT) dot_fused_kernel(int64_t n, int nb, int chunk, int k2, const double* __restrict__ a,
                                 const double* __restrict__ b,
                                 const double* __restrict__ a2, const double* __restrict__ b2,
                                 double* __restrict__ partial, double* __restrict__ out, double* __restrict__ out2,
                                 unsigned* __restrict__ tickets) {
  const int c = blockIdx.y, blk = blockIdx.x;
  const bool two = a2 != nullptr && c < k2;
  const int64_t off = (int64_t)c * n;
  const int64_t i0 = (int64_t)blk * chunk;
  const int64_t i1 = i0 + chunk < n ? i0 + chunk : n;
  __shared__ bool last;
  double v, v2;
  block_dots<DT>(off, i0, i1, a, b, a2, b2, two, v, v2);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      if (nb == 1) {  // one block per column: it holds the whole dot
        out[c] = v;
        if (two) out2[c] = v2;
        last = false;
      } else {
        partial[((int64_t)c * nb + blk) * 2] = v;
        partial[((int64_t)c * nb + blk) * 2 + 1] = v2;
        __threadfence();
        last = atomicAdd(&tickets[c], 1u) == (unsigned)(nb - 1);
      }
    }
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  const volatile double* pv = partial + (int64_t)c * nb * 2;
  double t = 0.0, t2 = 0.0;
  for (int i = threadIdx.x; i < nb; i += 32) {
    t += pv[2 * i];
    t2 += pv[2 * i + 1];
  }
  t = warp_sum(t);
  t2 = warp_sum(t2);
  if (threadIdx.x == 0) {
    out[c] = t;
    if (two) out2[c] = t2;
    tickets[c] = 0u;
  }
}

// block size of dot_fused_kernel (env KGP_DOT_THREADS: 256 | 512 | 1024)
int dot_threads() {
  static const int v = [] {
    const char* s = getenv("KGP_DOT_THREADS");
    const int t = s ? atoi(s) : 1024;
    return t >= 1024 ? 1024 : t >= 512 ? 512 : 256;
  }();
  return v;
}

template <class... A>
void launch_dot_fused(dim3 grid, cudaStream_t st, A... args) {
  switch (dot_threads()) {
    case 1024: dot_fused_kernel<1024><<<grid, 1024, 0, st>>>(args...); break;
    case 512: dot_fused_kernel<512><<<grid, 512, 0, st>>>(args...); break;
    default: dot_fused_kernel<256><<<grid, 256, 0, st>>>(args...); break;
  }
}

struct PcgState {
  double *x, *r, *z, *p, *ap;  // (k, n)
  double *rz, *ynorm, *alpha, *beta, *dots1, *dots2, *partial;
  unsigned* tickets;  // k zero-initialised counters for dot_fused_kernel
  int32_t* active;
  int32_t* status;  // [0] active count, [1] error code, [2] error column (min), [3] pad
  double* err_val;
};

// Columns [0, kpc) form group 1 (preconditioned when a preconditioner is given; tol1, cap it1),
// columns [kpc, k) group 2 (never preconditioned; tol2, cap it2): one operator application per
// iteration serves both, e.g. the w-solve and the probe solves of nlml_grad_iterative
// (gp.py:154-160) as Khat [p_w, P_Z]. Each column's recurrence is independent of the others.
struct PcgGroups {
  int kpc;
  int kz;      // leading columns whose z is M^-1 r (kpc, or k when the probes are preconditioned too)
  double tol1, tol2;
  int it1, it2;
  int stride;  // per-column stride of the alpha/beta arrays (max(it1, it2))
  __device__ double tol(int c) const { return c < kpc ? tol1 : tol2; }
  __device__ int cap(int c) const { return c < kpc ? it1 : it2; }
};

__global__ void pcg_init_kernel(int k, PcgGroups g, const double* ynorm_sq, double* ynorm, double* rel,
                                int32_t* active, int32_t* iters, int32_t* status) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0) {
    status[1] = 0;
    status[2] = 0x7fffffff;
  }
  if (c >= k) return;
  double yn = sqrt(ynorm_sq[c]);
  ynorm[c] = yn;
  double rl = yn > 0.0 ? 1.0 : 0.0;  // solver.py:150
  rel[c] = rl;
  int a = rl > g.tol(c) ? 1 : 0;
  active[c] = a;
  iters[c] = 0;
  if (a) atomicAdd(&status[0], 1);
}

// alpha step (solver.py:159-168) fused with x += alpha p; r -= alpha Ap on active columns:
// every block derives alpha_c = rz_c / pAp_c itself, block 0 of the column records it
__global__ void pcg_alpha_update_kernel(int64_t n, int k, int stride, const double* pap, const double* rz,
                                        const int32_t* active, const int32_t* iters, double* alphas, int32_t* status,
                                        double* err_val, const double* p, const double* ap, double* x, double* r) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  const double v = pap[c];
  if (!isfinite(v) || v <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      int old = atomicMin(&status[2], c);
      status[1] = KGP_ERR_BREAKDOWN;
      if (c <= old) err_val[0] = v;
    }
    return;
  }
  const double a = rz[c] / v;
  if (blockIdx.x == 0 && threadIdx.x == 0) alphas[(int64_t)c * stride + iters[c]] = a;
  const int64_t off = (int64_t)c * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[off + i] = fma(a, p[off + i], x[off + i]);
    r[off + i] = fma(-a, ap[off + i], r[off + i]);
  }
}

// beta step and freeze decision (solver.py:170-182)
// One block (k <= 1024). Also publishes (active count, error code, active count of group 1)
// of this iteration to hist[HIST * it], a host-mapped array the driver polls a few
// iterations behind the device.
__global__ void pcg_beta_kernel(int k, PcgGroups g, bool precond, const double* rr, const double* rzn,
                                double* rz, const double* ynorm, int32_t* active, int32_t* iters, double* beta,
                                double* betas, double* rel, int32_t* status, int32_t* it_counter,
                                volatile int32_t* hist) {
  int c = threadIdx.x;
  if (c == 0) {
    status[0] = 0;
    status[3] = 0;
  }
  __syncthreads();
  if (c < k && active[c]) {
    double v = rr[c];
    if (!isfinite(v)) {
      atomicMin(&status[2], c);
      status[1] = KGP_ERR_NUMERICAL;
    } else {
      double rn = (precond && c < g.kz) ? rzn[c] : v;
      double b = rn / rz[c];
      int it = iters[c];
      betas[(int64_t)c * g.stride + it] = b;
      iters[c] = it + 1;
      rz[c] = rn;
      double rl = sqrt(v) / ynorm[c];
      rel[c] = rl;
      beta[c] = b;
      if (rl <= g.tol(c) || it + 1 >= g.cap(c)) {  // converged, or this column's iteration cap
        active[c] = 0;
      } else {
        atomicAdd(&status[0], 1);
        if (c < g.kpc) atomicAdd(&status[3], 1);
      }
    }
  }
  __syncthreads();
  if (c == 0) {
    __threadfence();
    const int it = *it_counter;
    hist[HIST * it] = status[0];
    hist[HIST * it + 1] = status[1];
    hist[HIST * it + 2] = status[3];
    *it_counter = it + 1;
  }
}

// p = z + beta p on the still-active columns (z = r on the unpreconditioned group)
__global__ void pcg_update_p_kernel(int64_t n, int k, int kpc, const int32_t* active, const double* beta,
                                    const double* z, const double* r, double* p) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  const double b = beta[c];
  const int64_t off = (int64_t)c * n;
  const double* zc = (c < kpc ? z : r) + off;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[off + i] = fma(b, p[off + i], zc[i]);
}

__global__ void pcg_finish_kernel(int k, PcgGroups g, const double* rel, int32_t* conv) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < k) conv[c] = rel[c] <= g.tol(c) ? 1 : 0;
}

// ---------------------------------------------------------------- SLQ
// Implicit-shift QL on the symmetric tridiagonal (d, e), rotating only the first
// row z of the eigenvector matrix (element i of each array at [i * S]: the per-thread
// arrays of a block are interleaved in shared memory). Returns false if an eigenvalue
// does not converge in 60 sweeps. The rotation length sqrt(f^2 + g^2) is formed directly
// (hypot's rescaling only matters far outside the range of Lanczos coefficients; it is
// kept as the fallback there) and divided once.
__device__ __forceinline__ double rot_len(double f, double g) {
  const double r = sqrt(fma(f, f, g * g));
  return (r > 1e-150 && r < 1e150) ? r : hypot(f, g);
}

__device__ bool tridiag_ql_first_row(int m, double* d, double* e, double* z, int S) {
  for (int l = 0; l < m; ++l) {
    int sweeps = 0;
    while (true) {
      int mm = l;
      for (; mm < m - 1; ++mm) {
        const double dd = fabs(d[mm * S]) + fabs(d[(mm + 1) * S]);
        if (fabs(e[mm * S]) <= 2.2204460492503131e-16 * dd) break;
      }
      if (mm == l) break;
      if (++sweeps > 60) return false;
      const double dl = d[l * S];
      double g = (d[(l + 1) * S] - dl) / (2.0 * e[l * S]);
      double r = rot_len(g, 1.0);
      g = d[mm * S] - dl + e[l * S] / (g + copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      int i = mm - 1;
      bool deflated = false;
      double zi1 = z[mm * S];  // z[i + 1], carried in a register down the sweep
      for (; i >= l; --i) {
        const double ei = e[i * S];
        const double f = s * ei, b = c * ei;
        r = rot_len(f, g);
        e[(i + 1) * S] = r;
        if (r == 0.0) {  // split: the rotation underflowed
          d[(i + 1) * S] -= p;
          e[mm * S] = 0.0;
          deflated = true;
          break;
        }
        const double rinv = 1.0 / r;
        s = f * rinv;
        c = g * rinv;
        g = d[(i + 1) * S] - p;
        r = (d[i * S] - g) * s + 2.0 * c * b;
        p = s * r;
        d[(i + 1) * S] = g + p;
        g = c * r - b;
        const double zi = z[i * S];
        z[(i + 1) * S] = s * zi + c * zi1;
        zi1 = c * zi - s * zi1;
      }
      if (deflated) {
        z[(i + 1) * S] = zi1;
        continue;
      }
      z[l * S] = zi1;
      d[l * S] -= p;
      e[l * S] = g;
      e[mm * S] = 0.0;
    }
  }
  return true;
}

// One thread per probe. ws: nullptr = the per-thread arrays live in dynamic shared memory
// (3 * max_iter doubles per thread, interleaved); else a global scratch of the same layout.
__global__ void slq_kernel(int k, int max_iter, const double* __restrict__ alphas, const double* __restrict__ betas,
                           const int32_t* __restrict__ iters, const double* __restrict__ norms_sq,
                           double* __restrict__ ws, double* __restrict__ contrib, int32_t* __restrict__ status) {
  extern __shared__ double slq_smem[];
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  const int m = iters[c];
  if (m == 0) {  // zero-iteration probes contribute 0 but count (solver.py:253-255)
    contrib[c] = 0.0;
    return;
  }
  const int S = blockDim.x;
  double* base = ws ? ws + (size_t)blockIdx.x * blockDim.x * 3 * max_iter : slq_smem;
  double* d = base + threadIdx.x;
  double* e = d + (size_t)max_iter * S;
  double* z = e + (size_t)max_iter * S;
  const double* a = alphas + (int64_t)c * max_iter;
  const double* b = betas + (int64_t)c * max_iter;
  // solver.py:232-234: d_i = 1/a_i + b_{i-1}/a_{i-1}; e_i = sqrt(b_i)/a_i
  for (int i = 0; i < m; ++i) {
    d[i * S] = 1.0 / a[i] + (i > 0 ? b[i - 1] / a[i - 1] : 0.0);
    e[i * S] = (i < m - 1) ? sqrt(b[i]) / a[i] : 0.0;
    z[i * S] = (i == 0) ? 1.0 : 0.0;
  }
  if (!tridiag_ql_first_row(m, d, e, z, S)) {
    status[1] = KGP_ERR_NUMERICAL;
    contrib[c] = NAN;
    return;
  }
  double wmin = d[0], acc = 0.0;
  for (int i = 0; i < m; ++i) wmin = fmin(wmin, d[i * S]);
  if (!(wmin > 0.0)) {
    status[1] = KGP_ERR_NUMERICAL;
    atomicMax(&status[2], k - c);  // lowest failing column = k - status[2]
    contrib[c] = wmin;
    return;
  }
  for (int i = 0; i < m; ++i) acc += z[i * S] * z[i * S] * log(d[i * S]);
  contrib[c] = norms_sq[c] * acc;
}

int read_status(const int32_t* dev_status, int32_t* host4, cudaStream_t st) {
  KGP_CUDA(cudaMemcpyAsync(host4, dev_status, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost, st));
  KGP_CUDA(cudaStreamSynchronize(st));
  return KGP_OK;
}

}  // namespace

int col_dots(int64_t k, int64_t n, const double* a, const double* b, double* out, double* partial, cudaStream_t st) {
  int nb = (int)((n + DOT_CHUNK - 1) / DOT_CHUNK);
  dim3 g1(nb, (unsigned)k);
  dot_partial_kernel<<<g1, DOT_THREADS, 0, st>>>(n, nb, a, b, partial);
  KGP_LAUNCH("dot_partial_kernel");
  dot_final_kernel<<<(unsigned)k, 32, 0, st>>>((int)k, nb, partial, out);
  KGP_LAUNCH("dot_final_kernel");
  return KGP_OK;
}

// Device PCG state lives in the engine's workspace (not in the caller's buffers) so one
// captured CUDA graph of the iteration body can be replayed across calls. The body is
// captured once per (k, preconditioner, tol, max_iter) and launched with a look-ahead of
// kLookahead iterations: the host polls the per-iteration (active, error) history that
// pcg_beta_kernel writes into mapped host memory instead of synchronising every
// iteration. Iterations issued after convergence are no-ops (every update is masked by
// the per-column active flag), so results equal the synchronous loop's.
namespace {
constexpr int kLookahead = PCG_LOOKAHEAD;

struct PcgBuffers {
  PcgState S;
  double *x, *alphas, *betas, *rel;
  int32_t *iters, *it_counter;
};

// M^-1 on the first kpc columns: one handle for all of them, or one handle per column
// M^-1 on columns [0, kz): columns [0, kpc) by pcs.h (one handle, or one per column), columns
// [kpc, kz) (preconditioned probes) by pcs.tail (default h[0]), batched
int apply_pcs(const PcSet& pcs, int64_t kpc, int64_t kz, int64_t n, const double* r, double* z, cudaStream_t st) {
  int rc = KGP_OK;
  const int64_t head = kpc < kz ? kpc : kz;
  kgp_precond_s* tail = pcs.tail ? pcs.tail : pcs.h[0];
  if (pcs.count == 1 && tail == pcs.h[0]) return precond_apply_impl(pcs.h[0], kz, r, 1, n, z, 1, n, st);
  if (pcs.count == 1) {
    if (head > 0) rc = precond_apply_impl(pcs.h[0], head, r, 1, n, z, 1, n, st);
  } else {
    for (int64_t c = 0; c < head && !rc; ++c)
      rc = precond_apply_impl(pcs.h[c], 1, r + c * n, 1, n, z + c * n, 1, n, st);
  }
  if (!rc && kz > head) {
    if (pcs.probe_kz > 0 && pcs.count == kpc) {
      // per-class probe blocks (preconditioned-probe GPC): block c preconditioned by class c's handle
      for (int64_t c = 0; c < kpc && !rc; ++c) {
        const int64_t c0 = head + c * pcs.probe_kz;
        rc = precond_apply_impl(pcs.h[c], pcs.probe_kz, r + c0 * n, 1, n, z + c0 * n, 1, n, st);
      }
    } else {
      rc = precond_apply_impl(tail, kz - head, r + head * n, 1, n, z + head * n, 1, n, st);
    }
  }
  return rc;
}

int enqueue_iteration(kgp_engine_s* e, const PcSet& pcs, int64_t k, const PcgGroups& g, const PcgBuffers& B,
                      cudaStream_t st) {
  const bool pc = pcs.count > 0;
  const int64_t n = e->n;
  const PcgState& S = B.S;
  dim3 vgrid((unsigned)((n + 255) / 256 < 64 ? (n + 255) / 256 : 64), (unsigned)k);
  const int chunk = fused_chunk();
  const int nb = (int)((n + chunk - 1) / chunk);
  int rc = engine_matmul_impl(e, k, S.p, 1, n, S.ap, nullptr, nullptr, 1, n, st);
  if (rc) return rc;
  launch_dot_fused(dim3((unsigned)nb, (unsigned)k), st, n, nb, chunk, 0, S.p, S.ap, nullptr, nullptr, S.partial,
                   S.dots1, nullptr, S.tickets);
  KGP_LAUNCH("dot_fused_kernel");
  pcg_alpha_update_kernel<<<vgrid, 256, 0, st>>>(n, (int)k, g.stride, S.dots1, S.rz, S.active, B.iters, B.alphas,
                                                 S.status, S.err_val, S.p, S.ap, B.x, S.r);
  KGP_LAUNCH("pcg_alpha_update_kernel");
  if (pc && g.kz > 0) {  // M^-1 on the preconditioned columns only
    rc = apply_pcs(pcs, g.kpc, g.kz, n, S.r, S.z, st);
    if (rc) return rc;
  }
  // r.r on every column and r.z on the preconditioned ones, one launch
  launch_dot_fused(dim3((unsigned)nb, (unsigned)k), st, n, nb, chunk, pc ? g.kz : 0, S.r, S.r, pc ? S.r : nullptr,
                   pc ? S.z : nullptr, S.partial, S.dots1, S.dots2, S.tickets);
  KGP_LAUNCH("dot_fused_kernel");
  const int bt = (int)((k + 31) / 32 * 32);
  pcg_beta_kernel<<<1, bt, 0, st>>>((int)k, g, pc, S.dots1, S.dots2, S.rz, S.ynorm, S.active, B.iters,
                                      S.beta, B.betas, B.rel, S.status, B.it_counter, e->hist_dev);
  KGP_LAUNCH("pcg_beta_kernel");
  pcg_update_p_kernel<<<vgrid, 256, 0, st>>>(n, (int)k, pc ? g.kz : 0, S.active, S.beta, S.z, S.r, S.p);
  KGP_LAUNCH("pcg_update_p_kernel");
  return KGP_OK;
}

bool same_groups(const PcgGraph& c, int64_t k, const PcSet& pcs, const PcgGroups& g) {
  if (!c.exec || (int)c.pcs.size() != pcs.count || c.tail != pcs.tail || c.probe_kz != pcs.probe_kz) return false;
  for (int i = 0; i < pcs.count; ++i)
    if (c.pcs[i] != pcs.h[i]) return false;
  return c.k == k && c.kpc == g.kpc && c.kz == g.kz && c.tol1 == g.tol1 && c.tol2 == g.tol2 &&
         c.it1 == g.it1 && c.it2 == g.it2 && c.epoch == graph_epoch();
}

// returns the graph for this configuration, capturing it on first use
int pcg_graph(kgp_engine_s* e, const PcSet& pcs, int64_t k, const PcgGroups& g, const PcgBuffers& B,
              cudaGraphExec_t* out, int64_t* kernels) {
  for (auto& c : e->gcache)
    if (same_groups(c, k, pcs, g)) {
      *out = c.exec;
      *kernels = c.kernels;
      return KGP_OK;
    }
  // captured on the engine's private stream (the legacy default stream cannot be captured);
  // nothing is executed during capture, so no ordering with the caller's stream is needed.
  // Relaxed mode: a workspace the captured configuration needs for the first time is
  // allocated during the capture (cudaMalloc is refused in the stricter modes); graphs
  // captured before that allocation are retired by the epoch bump.
  cudaGraph_t graph = nullptr;
  const int64_t counted = kgp_launch_count();
  KGP_CUDA(cudaStreamBeginCapture(e->cstream, cudaStreamCaptureModeRelaxed));
  e->gate = B.S.status;  // status[0]: active columns after the previous iteration's beta
  int rc = enqueue_iteration(e, pcs, k, g, B, e->cstream);
  e->gate = nullptr;
  cudaError_t ce = cudaStreamEndCapture(e->cstream, &graph);
  count_launches(counted - kgp_launch_count());  // captured, not launched
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  KGP_CUDA(ce);
  size_t nodes = 0;
  cudaGraphGetNodes(graph, nullptr, &nodes);
  std::vector<cudaGraphNode_t> all(nodes);
  int64_t nkern = 0;
  if (nodes && cudaGraphGetNodes(graph, all.data(), &nodes) == cudaSuccess)
    for (auto nd : all) {
      cudaGraphNodeType t;
      if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++nkern;
    }
  cudaGraphExec_t exec = nullptr;
  ce = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  KGP_CUDA(ce);
  auto& slot = e->gcache[e->gnext];
  e->gnext = (e->gnext + 1) % (int)(sizeof(e->gcache) / sizeof(e->gcache[0]));
  if (slot.exec) cudaGraphExecDestroy(slot.exec);
  slot.exec = exec;
  slot.k = k;
  slot.pcs.assign(pcs.h, pcs.h + pcs.count);
  slot.tail = pcs.tail;
  slot.probe_kz = pcs.probe_kz;
  slot.kpc = g.kpc;
  slot.kz = g.kz;
  slot.tol1 = g.tol1;
  slot.tol2 = g.tol2;
  slot.it1 = g.it1;
  slot.it2 = g.it2;
  slot.epoch = graph_epoch();
  slot.kernels = nkern;
  *out = exec;
  *kernels = nkern;
  return KGP_OK;
}

int status_error(const PcgState& S, int code, int32_t col) {
  if (code == KGP_ERR_BREAKDOWN) {
    double v = 0.0;
    cudaMemcpy(&v, S.err_val, sizeof(double), cudaMemcpyDeviceToHost);
    set_error(KGP_ERR_BREAKDOWN, "p^T A p = %.17g in column %d; operator is not SPD", v, col);
    return KGP_ERR_BREAKDOWN;
  }
  set_error(KGP_ERR_NUMERICAL, "residual became non-finite during PCG");
  return KGP_ERR_NUMERICAL;
}
}  // namespace

int pcg_solve_impl(kgp_engine_s* e, kgp_precond_s* pc, int64_t k, const double* y, double tol, int max_iter,
                   double* x_out, double* alphas, double* betas, int32_t* iters, double* rel, int32_t* conv,
                   cudaStream_t st) {
  kgp_precond_s* one[1] = {pc};
  return pcg_grouped_impl(e, PcSet{one, pc ? 1 : 0}, k, k, y, tol, max_iter, tol, max_iter, x_out, alphas, betas,
                          iters, rel, conv, st, false);
}

int pcg_grouped_impl(kgp_engine_s* e, const PcSet& pcs, int64_t k, int64_t kpc, const double* y, double tol1,
                     int it1, double tol2, int it2, double* x_out, double* alphas, double* betas, int32_t* iters,
                     double* rel, int32_t* conv, cudaStream_t st, bool precond_all) {
  const int64_t n = e->n;
  const int nb = (int)((n + fused_chunk() - 1) / fused_chunk() + (n + DOT_CHUNK - 1) / DOT_CHUNK);
  KGP_REQUIRE(k <= 1024, KGP_ERR_INVALID, "pcg supports at most 1024 right-hand sides per call, got %lld",
              (long long)k);
  KGP_REQUIRE(kpc >= 0 && kpc <= k && it1 >= 1 && (kpc == k || it2 >= 1), KGP_ERR_INVALID, "bad column groups");
  KGP_REQUIRE(pcs.count <= 1 || pcs.count == kpc, KGP_ERR_INVALID,
              "need one preconditioner or one per preconditioned column (%d for %lld)", pcs.count, (long long)kpc);
  for (int i = 0; i < pcs.count; ++i)
    KGP_REQUIRE(pcs.h[i] != nullptr && pcs.h[i]->n == e->n, KGP_ERR_INVALID, "preconditioner %d missing or of wrong size", i);
  const bool pc = pcs.count > 0;
  KGP_REQUIRE(!precond_all || pcs.count == 1 || pcs.tail || (pcs.probe_kz > 0 && pcs.count == kpc &&
                                                              kpc + kpc * pcs.probe_kz == k),
              KGP_ERR_INVALID, "preconditioning every column needs one handle, a tail handle or per-class blocks");
  PcgGroups g{(int)kpc, 0, tol1, kpc < k ? tol2 : tol1, it1, kpc < k ? it2 : it1, 0};
  g.kz = pcs.count == 0 ? 0 : (precond_all ? (int)k : (int)kpc);
  if (kpc == 0) {
    g.tol1 = g.tol2;
    g.it1 = g.it2;
  }
  const int max_iter = g.it1 > g.it2 ? g.it1 : g.it2;
  g.stride = max_iter;
  // engine-owned state: r, p, ap, [z], x : (k, n); coefficient arrays; scalars
  const size_t vec = (size_t)k * n;
  const size_t coef = (size_t)k * max_iter;
  size_t bytes = sizeof(double) * (vec * (pc ? 5 : 4) + 2 * coef + (size_t)k * (9 + 2 * nb) + 8) +
                 sizeof(int32_t) * (3 * k + 16);
  int rc = e->ws.ensure(bytes);
  if (rc) return rc;
  if (e->hist_cap < max_iter + 1) {  // mapped host history: HIST ints per iteration
    if (e->hist_host) cudaFreeHost(e->hist_host);
    e->hist_host = nullptr;
    KGP_CUDA(cudaHostAlloc(&e->hist_host, sizeof(int32_t) * HIST * (max_iter + 1), cudaHostAllocMapped));
    KGP_CUDA(cudaHostGetDevicePointer((void**)&e->hist_dev, e->hist_host, 0));
    e->hist_cap = max_iter + 1;
    bump_graph_epoch();
  }
  double* base = e->ws.as<double>();
  PcgBuffers B{};
  PcgState& S = B.S;
  S.r = base;
  S.p = S.r + vec;
  S.ap = S.p + vec;
  B.x = S.ap + vec;
  S.x = B.x;
  S.z = pc ? B.x + vec : S.r;  // unpreconditioned: z aliases r (solver.py:195-199)
  double* sc = (pc ? S.z : B.x) + vec;
  B.alphas = sc;
  B.betas = sc + coef;
  sc += 2 * coef;
  S.rz = sc;
  S.ynorm = sc + k;
  S.alpha = sc + 2 * k;
  S.beta = sc + 3 * k;
  S.dots1 = sc + 4 * k;
  S.dots2 = sc + 5 * k;
  S.err_val = sc + 6 * k;
  B.rel = sc + 7 * k;
  S.partial = sc + 8 * k;
  S.active = reinterpret_cast<int32_t*>(S.partial + (size_t)2 * k * nb + 8);
  S.status = S.active + k;  // 4 ints
  B.iters = S.status + 4;
  B.it_counter = B.iters + k;
  S.tickets = reinterpret_cast<unsigned*>(B.it_counter + 4);

  int32_t* hstatus = e->hstatus;
  const unsigned kb = (unsigned)((k + 127) / 128);

  KGP_CUDA(cudaMemsetAsync(B.x, 0, sizeof(double) * vec, st));
  KGP_CUDA(cudaMemcpyAsync(S.r, y, sizeof(double) * vec, cudaMemcpyDeviceToDevice, st));
  KGP_CUDA(cudaMemsetAsync(S.status, 0, sizeof(int32_t) * 4, st));
  KGP_CUDA(cudaMemsetAsync(B.it_counter, 0, sizeof(int32_t), st));
  KGP_CUDA(cudaMemsetAsync(S.tickets, 0, sizeof(unsigned) * k, st));
  KGP_CUDA(cudaMemsetAsync(B.alphas, 0, sizeof(double) * 2 * coef, st));
  rc = col_dots(k, n, S.r, S.r, S.dots1, S.partial, st);
  if (rc) return rc;
  pcg_init_kernel<<<kb, 128, 0, st>>>((int)k, g, S.dots1, S.ynorm, B.rel, S.active, B.iters, S.status);
  KGP_LAUNCH("pcg_init_kernel");
  rc = read_status(S.status, hstatus, st);
  if (rc) return rc;
  if (hstatus[0] > 0) {
    const int64_t kz = g.kz;  // columns whose z is M^-1 r
    if (kz > 0) {
      rc = apply_pcs(pcs, g.kpc, kz, n, S.r, S.z, st);
      if (rc) return rc;
      KGP_CUDA(cudaMemcpyAsync(S.p, S.z, sizeof(double) * kz * n, cudaMemcpyDeviceToDevice, st));
      rc = col_dots(kz, n, S.r, S.z, S.rz, S.partial, st);
      if (rc) return rc;
    }
    if (kz < k) {
      KGP_CUDA(cudaMemcpyAsync(S.p + kz * n, S.r + kz * n, sizeof(double) * (k - kz) * n, cudaMemcpyDeviceToDevice,
                               st));
      rc = col_dots(k - kz, n, S.r + kz * n, S.r + kz * n, S.rz + kz, S.partial, st);
      if (rc) return rc;
    }
    // iteration 0 uncaptured: it also performs every lazy allocation / first-launch setup
    rc = enqueue_iteration(e, pcs, k, g, B, st);
    if (rc) return rc;
    KGP_CUDA(cudaStreamSynchronize(st));
    volatile int32_t* H = e->hist_host;
    if (H[1]) return status_error(S, H[1], 0);
    bool done = (H[0] == 0);
    if (!done && max_iter > 1) {
      cudaGraphExec_t exec = nullptr;
      int64_t gk = 0;
      rc = pcg_graph(e, pcs, k, g, B, &exec, &gk);
      if (rc) return rc;
      // once every group-2 column has stopped (its cap, or converged), the remaining
      // iterations run a graph over the group-1 prefix [0, kpc) only: the state is column-major
      // with group 1 first, so the same buffers serve both graphs
      bool narrow = !(kpc > 0 && kpc < k);
      auto go_narrow = [&]() -> int {
        PcgGroups gn = g;
        gn.kz = g.kz < g.kpc ? g.kz : g.kpc;
        int rc2 = pcg_graph(e, pcs, kpc, gn, B, &exec, &gk);
        narrow = true;
        return rc2;
      };
      int launched = 1, checked = 1;
      while (launched < max_iter && !done) {
        KGP_CUDA(cudaGraphLaunch(exec, st));
        count_launches(gk);
        KGP_CUDA(cudaEventRecord(e->events[launched % kLookahead], st));
        ++launched;
        // every group-2 column stops by its cap it2 at the latest: after it2 iterations the
        // narrow graph is exact without waiting for the (look-ahead delayed) history
        if (!narrow && launched >= g.it2) {
          rc = go_narrow();
          if (rc) return rc;
        }
        if (launched - checked >= kLookahead) {
          KGP_CUDA(cudaEventSynchronize(e->events[checked % kLookahead]));
          if (H[HIST * checked + 1]) {
            KGP_CUDA(cudaStreamSynchronize(st));
            KGP_CUDA(cudaMemcpy(hstatus, S.status, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost));
            return status_error(S, H[HIST * checked + 1], hstatus[2]);
          }
          done = (H[HIST * checked] == 0);
          if (!done && !narrow && H[HIST * checked] == H[HIST * checked + 2]) {
            rc = go_narrow();
            if (rc) return rc;
          }
          ++checked;
        }
      }
      KGP_CUDA(cudaStreamSynchronize(st));
      for (; checked < launched; ++checked) {
        if (H[HIST * checked + 1]) {
          KGP_CUDA(cudaMemcpy(hstatus, S.status, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost));
          return status_error(S, H[HIST * checked + 1], hstatus[2]);
        }
        if (H[HIST * checked] == 0) break;
      }
    }
  }
  pcg_finish_kernel<<<kb, 128, 0, st>>>((int)k, g, B.rel, conv);
  KGP_LAUNCH("pcg_finish_kernel");
  KGP_CUDA(cudaMemcpyAsync(x_out, B.x, sizeof(double) * vec, cudaMemcpyDeviceToDevice, st));
  KGP_CUDA(cudaMemcpyAsync(alphas, B.alphas, sizeof(double) * coef, cudaMemcpyDeviceToDevice, st));
  KGP_CUDA(cudaMemcpyAsync(betas, B.betas, sizeof(double) * coef, cudaMemcpyDeviceToDevice, st));
  KGP_CUDA(cudaMemcpyAsync(iters, B.iters, sizeof(int32_t) * k, cudaMemcpyDeviceToDevice, st));
  KGP_CUDA(cudaMemcpyAsync(rel, B.rel, sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
  KGP_CUDA(cudaStreamSynchronize(st));
  return KGP_OK;
}

int slq_impl(int64_t k, int max_iter, const double* alphas, const double* betas, const int32_t* iters,
             const double* norms_sq, double* logdet, cudaStream_t st) {
  static thread_local DevBuf ws;  // persistent: cudaMalloc/cudaFree per call would serialise the device
  // per-thread arrays in shared memory when a block of >= 8 probes fits in 160 KB
  const size_t per_thread = sizeof(double) * 3 * (size_t)max_iter;
  const size_t smem_cap = 160 * 1024;
  int tpb = (int)(smem_cap / per_thread < 64 ? smem_cap / per_thread : 64);
  const bool in_smem = tpb >= 8 && getenv("KGP_SLQ_GLOBAL") == nullptr;
  if (!in_smem) tpb = 64;
  if (tpb > k) tpb = (int)((k + 7) / 8 * 8);
  const unsigned blocks = (unsigned)((k + tpb - 1) / tpb);
  const size_t scratch = in_smem ? 0 : (size_t)blocks * tpb * 3 * max_iter;
  int rc = ws.ensure(sizeof(double) * (scratch + k) + 64);
  if (rc) return rc;
  double* contrib = ws.as<double>() + scratch;
  int32_t* status = reinterpret_cast<int32_t*>(contrib + k);
  KGP_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * 4, st));
  const size_t smem = in_smem ? per_thread * tpb : 0;
  if (smem > 48 * 1024)
    KGP_CUDA(cudaFuncSetAttribute(slq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  slq_kernel<<<blocks, tpb, smem, st>>>((int)k, max_iter, alphas, betas, iters, norms_sq,
                                        in_smem ? nullptr : ws.as<double>(), contrib, status);
  KGP_LAUNCH("slq_kernel");
  std::vector<double> h(k);
  int32_t hs[4];
  KGP_CUDA(cudaMemcpyAsync(h.data(), contrib, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
  KGP_CUDA(cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st));
  KGP_CUDA(cudaStreamSynchronize(st));
  if (hs[1] == KGP_ERR_NUMERICAL) {
    const int64_t col = hs[2] > 0 ? k - hs[2] : -1;
    double w = (col >= 0 && col < k) ? h[col] : NAN;
    set_error(KGP_ERR_NUMERICAL, "nonpositive Ritz value %.17g; operator is not SPD or CG broke down", w);
    return KGP_ERR_NUMERICAL;
  }
  double total = 0.0;  // probe order, as solver.py:253-265
  for (int64_t c = 0; c < k; ++c) total += h[c];
  *logdet = total / (double)k;
  return KGP_OK;
}

// nlml_grad_iterative (gp.py:133-179) for C independent right-hand sides sharing the
// kernel hyperparameters: C = 1 is GP regression; C > 1 is the Dirichlet GP
// classification of gpc.py (class c: Khat + diag(dn_c), target y_c). Loss and gradient
// are sums over the classes.
// pp (preconditioned probes, C = 1, one handle M): the probes are draws z ~ N(0, M); the
// probe solves are preconditioned by M, SLQ then estimates log|M^-1/2 Khat M^-1/2| with
// |M^-1/2 z|^2 = z^T M^-1 z as the quadrature weights, loss adds logdet_m = log|M|, and the
// trace estimator uses E[(M^-1 z)^T dK (Khat^-1 z)] = tr(Khat^-1 dK).
static int nlml_impl(kgp_engine_s* e, const PcSet& pcs, int64_t C, const double* y, int64_t k_z,
                     const double* probes, double tol, int32_t max_iter, double probe_tol, int32_t probe_max_iter,
                     double* out, int32_t* out_converged, cudaStream_t st, bool pp = false, double logdet_m = 0.0) {
  const int64_t n = e->n;
  const int64_t kv = C * (1 + k_z);
  const int nb = (int)((n + DOT_CHUNK - 1) / DOT_CHUNK);
  const int32_t pmax = probe_max_iter > 0 ? probe_max_iter : max_iter;
  const int32_t wide = pmax > max_iter ? pmax : max_iter;  // per-column stride of the coefficient arrays
  // workspace: V = [y_1..y_C, Z_1..Z_C] (kv, n); U = [w, u]; dV_l, dV_f; traces; scalars
  size_t vec = (size_t)kv * n;
  size_t bytes = sizeof(double) * (4 * vec + 2 * (size_t)kv * wide + 4 * kv + (size_t)kv * nb + 16) +
                 sizeof(int32_t) * (4 * kv + 8);
  DevBuf& ws = e->ws_nlml;  // persistent per engine (a training loop reuses it every step)
  int rc = ws.ensure(bytes);
  if (rc) return rc;
  double* V = ws.as<double>();
  double* U = V + vec;
  double* dL = U + vec;
  double* dF = dL + vec;
  double* alphas = dF + vec;
  double* betas = alphas + (size_t)kv * wide;
  double* rel = betas + (size_t)kv * wide;
  double* dots = rel + kv;
  double* nz2 = dots + kv;
  double* partial = nz2 + kv;
  int32_t* iters = reinterpret_cast<int32_t*>(partial + (size_t)kv * nb + 8);
  int32_t* conv = iters + kv;

  // (1)+(2) w = PCG(Khat, M, y, tol) and u = CG(Khat, Z, probe_tol) (gp.py:154-160) as ONE
  // grouped solve: every iteration applies Khat once to [p_w, P_Z] (the north star's
  // Khat [y, Z]); the C target columns are preconditioned, the probe columns are not, so
  // their coefficients rebuild the Lanczos tridiagonals of Khat itself.
  KGP_CUDA(cudaMemcpyAsync(V, y, sizeof(double) * C * n, cudaMemcpyDeviceToDevice, st));
  KGP_CUDA(cudaMemcpyAsync(V + C * n, probes, sizeof(double) * C * k_z * n, cudaMemcpyDeviceToDevice, st));
  rc = pcg_grouped_impl(e, pcs, kv, C, V, tol, max_iter, probe_tol, pmax, U, alphas, betas, iters, rel, conv, st,
                        pp);
  if (rc) return rc;
  // (3) log|Khat_c| by SLQ over each class's probe traces
  double* Z = V + C * n;
  if (pp) {  // M^-1 Z (into dL as scratch), weights z^T M^-1 z, then V's probe rows := M^-1 Z
    if (C > 1) {  // class c's probes by class c's preconditioner
      for (int64_t c = 0; c < C; ++c) {
        rc = precond_apply_impl(pcs.count == C ? pcs.h[c] : pcs.h[0], k_z, Z + c * k_z * n, 1, n,
                                dL + c * k_z * n, 1, n, st);
        if (rc) return rc;
      }
    } else {
      rc = precond_apply_impl(pcs.tail ? pcs.tail : pcs.h[0], k_z, Z, 1, n, dL, 1, n, st);
      if (rc) return rc;
    }
    rc = col_dots(C * k_z, n, Z, dL, nz2, partial, st);
    if (rc) return rc;
    KGP_CUDA(cudaMemcpyAsync(Z, dL, sizeof(double) * C * k_z * n, cudaMemcpyDeviceToDevice, st));
  } else {
    rc = col_dots(C * k_z, n, Z, Z, nz2, partial, st);
    if (rc) return rc;
  }
  double logdet = 0.0;
  for (int64_t c = 0; c < C; ++c) {
    double ld = 0.0;
    const size_t off = (size_t)(C + c * k_z) * wide;
    rc = slq_impl(k_z, wide, alphas + off, betas + off, iters + C + c * k_z, nz2 + c * k_z, &ld, st);
    if (rc) return rc;
    logdet += ld;
  }
  // (4) loss = 1/2 (y.w + logdet + n log 2 pi), summed over the classes
  rc = col_dots(C, n, y, U, dots, partial, st);
  if (rc) return rc;
  std::vector<double> hd(kv);
  KGP_CUDA(cudaMemcpyAsync(hd.data(), dots, sizeof(double) * C, cudaMemcpyDeviceToHost, st));
  KGP_CUDA(cudaStreamSynchronize(st));
  double yw = 0.0;
  for (int64_t c = 0; c < C; ++c) yw += hd[c];
  // (5) one fused derivative pass over V = [w, Z] (the diagonal is data: no derivative term)
  KGP_CUDA(cudaMemcpyAsync(V, U, sizeof(double) * C * n, cudaMemcpyDeviceToDevice, st));
  rc = engine_matmul_impl(e, kv, V, 1, n, nullptr, dL, dF, 1, n, st);
  if (rc) return rc;
  double grads[3];
  const double* dV[3] = {dL, dF, V};  // Theta.L, Theta.F, Theta.S (dKhat/ds = I, kmat.py:157-158)
  for (int th = 0; th < 3; ++th) {
    // column dots of [w, u] against dV columns: quad from the targets, trace from the probes
    rc = col_dots(kv, n, U, dV[th], dots, partial, st);
    if (rc) return rc;
    KGP_CUDA(cudaMemcpyAsync(hd.data(), dots, sizeof(double) * kv, cudaMemcpyDeviceToHost, st));
    KGP_CUDA(cudaStreamSynchronize(st));
    double g = 0.0;
    for (int64_t c = 0; c < C; ++c) {
      double tr = 0.0;
      for (int64_t j = 0; j < k_z; ++j) tr += hd[C + c * k_z + j];
      g += 0.5 * (-hd[c] + tr / (double)k_z);
    }
    grads[th] = g;
  }
  std::vector<int32_t> hc(kv);
  KGP_CUDA(cudaMemcpyAsync(hc.data(), conv, sizeof(int32_t) * kv, cudaMemcpyDeviceToHost, st));
  KGP_CUDA(cudaStreamSynchronize(st));
  int ok = 1;
  for (int64_t c = 0; c < kv; ++c) ok &= hc[c] ? 1 : 0;
  const double LOG_2PI = 1.8378770664093453;
  out[0] = 0.5 * (yw + logdet + logdet_m + (double)(C * n) * LOG_2PI);
  out[1] = grads[0];
  out[2] = grads[1];
  out[3] = grads[2];
  *out_converged = ok;
  return KGP_OK;
}

}  // namespace kgp

using namespace kgp;

extern "C" int kgp_nlml_grad(kgp_engine* e, kgp_precond* p, const double* y, int64_t k_z, const double* probes,
                             double tol, int32_t max_iter, double probe_tol, int32_t probe_max_iter, double* out,
                             int32_t* out_converged, void* stream) {
  KGP_REQUIRE(e != nullptr && e->magic == ENGINE_MAGIC, KGP_ERR_STATE, "invalid engine handle");
  KGP_REQUIRE(p == nullptr || p->magic == PRECOND_MAGIC, KGP_ERR_STATE, "invalid preconditioner handle");
  KGP_REQUIRE(k_z >= 1 && max_iter >= 1 && tol >= 0.0 && probe_tol >= 0.0, KGP_ERR_INVALID, "bad solver arguments");
  KGP_REQUIRE(out != nullptr && out_converged != nullptr, KGP_ERR_INVALID, "NULL output pointer");
  KGP_REQUIRE(e->dn_classes == 0, KGP_ERR_INVALID, "engine has a per-class diagonal; use kgp_gpc_nlml_grad");
  KGP_CUDA(cudaSetDevice(e->device));
  kgp_precond_s* one[1] = {p};
  return nlml_impl(e, PcSet{one, p ? 1 : 0}, 1, y, k_z, probes, tol, max_iter, probe_tol, probe_max_iter, out,
                   out_converged, (cudaStream_t)stream);
}

extern "C" int kgp_gpc_nlml_grad(kgp_engine* e, int classes, kgp_precond* const* pcs, int npcs, const double* dn,
                                 const double* y, int64_t k_z, const double* probes, double tol, int32_t max_iter,
                                 double probe_tol, int32_t probe_max_iter, double* out, int32_t* out_converged,
                                 void* stream) {
  KGP_REQUIRE(e != nullptr && e->magic == ENGINE_MAGIC, KGP_ERR_STATE, "invalid engine handle");
  KGP_REQUIRE(classes >= 1 && (npcs == 0 || npcs == 1 || npcs == classes), KGP_ERR_INVALID,
              "need classes >= 1 and 0, 1 or `classes` preconditioners");
  KGP_REQUIRE(npcs == 0 || pcs != nullptr, KGP_ERR_INVALID, "NULL preconditioner array");
  for (int i = 0; i < npcs; ++i)
    KGP_REQUIRE(pcs[i] != nullptr && pcs[i]->magic == PRECOND_MAGIC, KGP_ERR_STATE, "invalid preconditioner handle");
  KGP_REQUIRE(k_z >= 1 && max_iter >= 1 && tol >= 0.0 && probe_tol >= 0.0, KGP_ERR_INVALID, "bad solver arguments");
  KGP_REQUIRE(dn != nullptr && y != nullptr && probes != nullptr, KGP_ERR_INVALID, "NULL input pointer");
  KGP_REQUIRE(out != nullptr && out_converged != nullptr, KGP_ERR_INVALID, "NULL output pointer");
  KGP_REQUIRE(e->row0 == 0 && e->nrows == e->n, KGP_ERR_INVALID, "kgp_gpc_nlml_grad needs an unpartitioned engine");
  const int64_t kv = (int64_t)classes * (1 + k_z);
  std::vector<int32_t> map(kv);
  for (int64_t c = 0; c < kv; ++c) map[c] = (int32_t)(c < classes ? c : (c - classes) / k_z);
  int rc = kgp_engine_set_diag(e, classes, dn, kv, map.data(), stream);
  if (rc) return rc;
  rc = nlml_impl(e, PcSet{pcs, npcs}, classes, y, k_z, probes, tol, max_iter, probe_tol, probe_max_iter, out,
                 out_converged, (cudaStream_t)stream);
  kgp_engine_set_diag(e, 0, nullptr, 0, nullptr, stream);
  return rc;
}

extern "C" int kgp_gpc_nlml_grad_pp(kgp_engine* e, int classes, kgp_precond* const* pcs, const double* dn,
                                    const double* y, int64_t k_z, const double* probes, double logdet_m, double tol,
                                    int32_t max_iter, double probe_tol, int32_t probe_max_iter, double* out,
                                    int32_t* out_converged, void* stream) {
  KGP_REQUIRE(e != nullptr && e->magic == ENGINE_MAGIC, KGP_ERR_STATE, "invalid engine handle");
  KGP_REQUIRE(classes >= 1 && pcs != nullptr, KGP_ERR_INVALID, "need classes >= 1 and one preconditioner per class");
  for (int i = 0; i < classes; ++i)
    KGP_REQUIRE(pcs[i] != nullptr && pcs[i]->magic == PRECOND_MAGIC, KGP_ERR_STATE, "invalid preconditioner handle");
  KGP_REQUIRE(k_z >= 1 && max_iter >= 1 && tol >= 0.0 && probe_tol >= 0.0, KGP_ERR_INVALID, "bad solver arguments");
  KGP_REQUIRE(dn != nullptr && y != nullptr && probes != nullptr, KGP_ERR_INVALID, "NULL input pointer");
  KGP_REQUIRE(out != nullptr && out_converged != nullptr, KGP_ERR_INVALID, "NULL output pointer");
  KGP_REQUIRE(e->row0 == 0 && e->nrows == e->n, KGP_ERR_INVALID, "needs an unpartitioned engine");
  const int64_t kv = (int64_t)classes * (1 + k_z);
  std::vector<int32_t> map(kv);
  for (int64_t c = 0; c < kv; ++c) map[c] = (int32_t)(c < classes ? c : (c - classes) / k_z);
  int rc = kgp_engine_set_diag(e, classes, dn, kv, map.data(), stream);
  if (rc) return rc;
  PcSet set{pcs, classes};
  set.probe_kz = k_z;
  rc = nlml_impl(e, set, classes, y, k_z, probes, tol, max_iter, probe_tol, probe_max_iter, out, out_converged,
                 (cudaStream_t)stream, true, logdet_m);
  kgp_engine_set_diag(e, 0, nullptr, 0, nullptr, stream);
  return rc;
}

extern "C" int kgp_pcg_grouped(kgp_engine* e, kgp_precond* const* pcs, int npcs, int64_t k, int64_t kpc,
                               const double* y, double tol1, int32_t it1, double tol2, int32_t it2, double* x_out,
                               double* alphas, double* betas, int32_t* iters, double* rel, int32_t* converged,
                               void* stream) {
  KGP_REQUIRE(e != nullptr && e->magic == ENGINE_MAGIC, KGP_ERR_STATE, "invalid engine handle");
  KGP_REQUIRE(npcs >= 0 && (npcs == 0 || pcs != nullptr), KGP_ERR_INVALID, "bad preconditioner array");
  for (int i = 0; i < npcs; ++i)
    KGP_REQUIRE(pcs[i] != nullptr && pcs[i]->magic == PRECOND_MAGIC, KGP_ERR_STATE, "invalid preconditioner handle");
  KGP_REQUIRE(k >= 1 && tol1 >= 0.0 && tol2 >= 0.0, KGP_ERR_INVALID, "bad solver arguments");
  KGP_REQUIRE(e->row0 == 0 && e->nrows == e->n, KGP_ERR_INVALID, "kgp_pcg_grouped needs an unpartitioned engine");
  KGP_CUDA(cudaSetDevice(e->device));
  return pcg_grouped_impl(e, PcSet{pcs, npcs}, k, kpc, y, tol1, it1, tol2, it2, x_out, alphas, betas, iters, rel,
                          converged, (cudaStream_t)stream, false);
}

extern "C" int kgp_nlml_grad_pp(kgp_engine* e, kgp_precond* p_w, kgp_precond* p, const double* y, int64_t k_z,
                                const double* probes, double logdet_m, double tol, int32_t max_iter, double probe_tol,
                                int32_t probe_max_iter, double* out, int32_t* out_converged, void* stream) {
  KGP_REQUIRE(e != nullptr && e->magic == ENGINE_MAGIC, KGP_ERR_STATE, "invalid engine handle");
  KGP_REQUIRE(p != nullptr && p->magic == PRECOND_MAGIC, KGP_ERR_STATE, "preconditioned probes need a preconditioner");
  KGP_REQUIRE(p_w == nullptr || p_w->magic == PRECOND_MAGIC, KGP_ERR_STATE, "invalid w-solve preconditioner");
  KGP_REQUIRE(k_z >= 1 && max_iter >= 1 && tol >= 0.0 && probe_tol >= 0.0, KGP_ERR_INVALID, "bad solver arguments");
  KGP_REQUIRE(out != nullptr && out_converged != nullptr, KGP_ERR_INVALID, "NULL output pointer");
  KGP_REQUIRE(e->dn_classes == 0, KGP_ERR_INVALID, "engine has a per-class diagonal");
  KGP_REQUIRE(p->n == e->n && (p_w == nullptr || p_w->n == e->n), KGP_ERR_INVALID, "preconditioner size mismatch");
  KGP_CUDA(cudaSetDevice(e->device));
  kgp_precond_s* one[1] = {p_w ? p_w : p};
  PcSet pcs{one, 1};
  pcs.tail = p;
  return nlml_impl(e, pcs, 1, y, k_z, probes, tol, max_iter, probe_tol, probe_max_iter, out, out_converged,
                   (cudaStream_t)stream, true, logdet_m);
}
