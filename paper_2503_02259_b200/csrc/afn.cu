// AFN (adaptive factorized Nystrom) preconditioner on the device.
//
// The north star's PCG preconditioner: "landmark Cholesky solve plus sparse FSAI
// factor matvec". The reference replaces AFN by its Nystrom preconditioner
// (SPEC.md:17, 219-227), so there is no reference code path here; the numpy
// statement in tests/afn_ref.py is what these kernels are checked against.
//
// With landmarks X1 (m points) ordered first and the rest X2 (n2 points) after:
//   Khat = [K11 K12; K21 K22] = [I 0; W L^-1 I] [K11 0; 0 S] [I L^-T W^T; 0 I]
//   K11 = L L^T,  W = K21 L^-T (n2 x m),  S = K22 - W W^T (Schur complement)
// AFN keeps the landmark block exact and replaces S^-1 by a factorized sparse
// approximate inverse G^T G (G lower triangular, row i supported on i and its npt
// nearest earlier points of X2). Then
//   M^-1 b = [L^-T (y1 - W^T u2); u2],   y1 = L^-1 b1,   u2 = G^T G (b2 - W y1)
// i.e. per application: two tall-skinny fp64 GEMMs against W (HBM-bound, W is
// read twice), two small GEMMs against L^-1, one ELL and one CSR sparse product.
//
// Build kernels here: the earlier-point k-nearest-neighbour search that fixes the
// FSAI pattern, and one CTA per FSAI row that forms S_PP = Khat_PP - W_P W_P^T in
// shared memory, factors it and back-solves L^T z = e_last (z is row i of G:
// S_PP g = e_i scaled so that (G S G^T)_ii = 1). The dense factor work (K11
// Cholesky, W) is cuSOLVER/cuBLAS through torch on the host side (precond.py).
#include <math.h>

#include <vector>

#include <stdlib.h>

#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

// ------------------------------------------------------------------ k nearest earlier points
constexpr int KNN_T = 128;
constexpr int KNN_MAX = 64;         // FSAI pattern (earlier points)
constexpr int KNN_MAX_CROSS = 128;  // local predictive variance neighbourhoods

// PREV: queries are the candidates themselves (xq == x) and only j < i count (FSAI pattern);
// otherwise every candidate counts (nearest training points of test points).
template <int D, bool PREV, int MAXK = KNN_MAX>
__global__ void __launch_bounds__(KNN_T) knn_kernel(int64_t nq, const double* __restrict__ xq, int64_t nx,
                                                    const double* __restrict__ x, int npt, int64_t* __restrict__ out) {
  __shared__ double xs[KNN_T * D];
  const int64_t i = (int64_t)blockIdx.x * KNN_T + threadIdx.x;
  double q[D];
#pragma unroll
  for (int c = 0; c < D; ++c) q[c] = i < nq ? xq[i * D + c] : 0.0;
  double bd[MAXK];
  int64_t bj[MAXK];
  int cnt = 0;
  int64_t last = nx;
  if (PREV) last = (int64_t)(blockIdx.x + 1) * KNN_T < nx ? (int64_t)(blockIdx.x + 1) * KNN_T : nx;
  for (int64_t j0 = 0; j0 < last; j0 += KNN_T) {
    __syncthreads();
    for (int e = threadIdx.x; e < KNN_T * D; e += KNN_T) {
      const int64_t g = j0 * D + e;
      xs[e] = g < nx * D ? x[g] : 0.0;
    }
    __syncthreads();
    int64_t lim = PREV ? i - j0 : nx - j0;  // PREV: candidates j < i
    if (lim > KNN_T) lim = KNN_T;
    if (!PREV && i >= nq) lim = 0;
    for (int t = 0; t < lim; ++t) {
      double r = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double df = q[c] - xs[t * D + c];
        r = fma(df, df, r);
      }
      if (cnt < npt || r < bd[cnt - 1]) {  // strict: equal distances keep the lower j
        int p = cnt < npt ? cnt : npt - 1;
        while (p > 0 && bd[p - 1] > r) {
          bd[p] = bd[p - 1];
          bj[p] = bj[p - 1];
          --p;
        }
        bd[p] = r;
        bj[p] = j0 + t;
        if (cnt < npt) ++cnt;
      }
    }
  }
  if (i >= nq) return;
  for (int t = 0; t < npt; ++t) out[i * npt + t] = t < cnt ? bj[t] : -1;
}

// ------------------------------------------------------------------ FSAI rows
constexpr int FS_T = 128;
constexpr int FS_KC = 32;            // W columns per shared-memory chunk
constexpr int FS_MAXM = KNN_MAX + 1; // pattern size bound
constexpr int FS_MAXE = (FS_MAXM * (FS_MAXM + 1) / 2 + FS_T - 1) / FS_T;

struct FsaiSmem {
  double S[FS_MAXM * FS_MAXM];
  double Wc[FS_MAXM * (FS_KC + 1)];
  double xs[FS_MAXM * 16];
  double z[FS_MAXM];
  int idx[FS_MAXM];
  int m;
  int fail;
};

template <int KT>
__global__ void __launch_bounds__(FS_T) fsai_kernel(int64_t n2, int d, const double* __restrict__ x2, double l,
                                                    double f2, double s, int64_t mw, const double* __restrict__ w,
                                                    int npt, const int64_t* __restrict__ nbr,
                                                    const double* __restrict__ dshift,
                                                    double* __restrict__ gval, int32_t* __restrict__ gcol,
                                                    int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FsaiSmem& sm = *reinterpret_cast<FsaiSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int64_t i = blockIdx.x;
  if (tid == 0) {
    int m = 0;
    for (int t = 0; t < npt; ++t) {
      const int64_t j = nbr[i * npt + t];
      if (j >= 0) sm.idx[m++] = (int)j;
    }
    sm.idx[m++] = (int)i;
    sm.m = m;
    sm.fail = 0;
  }
  __syncthreads();
  const int m = sm.m;
  for (int e = tid; e < m * d; e += FS_T) sm.xs[e] = x2[(int64_t)sm.idx[e / d] * d + e % d];
  __syncthreads();
  // S_PP = f^2 kappa(x_P, x_P) + s I (lower triangle incl. diagonal)
  for (int e = tid; e < m * m; e += FS_T) {
    const int a = e / m, b = e % m;
    if (b > a) continue;
    double r2 = 0.0;
    for (int c = 0; c < d; ++c) {
      const double df = sm.xs[a * d + c] - sm.xs[b * d + c];
      r2 = fma(df, df, r2);
    }
    sm.S[a * m + b] = f2 * kappa64<KT>(r2, l) + (a == b ? s + (dshift ? dshift[sm.idx[a]] : 0.0) : 0.0);
  }
  // - W_P W_P^T, accumulated over the m_w landmark columns in chunks
  const int nent = m * (m + 1) / 2;
  int ea[FS_MAXE], eb[FS_MAXE];
  double acc[FS_MAXE];
#pragma unroll
  for (int t = 0; t < FS_MAXE; ++t) {
    const int e = tid + FS_T * t;
    int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (a * (a + 1) / 2 > e) --a;
    while ((a + 1) * (a + 2) / 2 <= e) ++a;
    ea[t] = a;
    eb[t] = e - a * (a + 1) / 2;
    acc[t] = 0.0;
  }
  for (int64_t q0 = 0; q0 < mw; q0 += FS_KC) {
    __syncthreads();
    for (int e = tid; e < m * FS_KC; e += FS_T) {
      const int a = e / FS_KC, q = e % FS_KC;
      sm.Wc[a * (FS_KC + 1) + q] = q0 + q < mw ? w[(int64_t)sm.idx[a] * mw + q0 + q] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < FS_MAXE; ++t) {
      if (tid + FS_T * t < nent) {
        const double* wa = sm.Wc + ea[t] * (FS_KC + 1);
        const double* wb = sm.Wc + eb[t] * (FS_KC + 1);
        double v = acc[t];
#pragma unroll 8
        for (int q = 0; q < FS_KC; ++q) v = fma(wa[q], wb[q], v);
        acc[t] = v;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < FS_MAXE; ++t)
    if (tid + FS_T * t < nent) sm.S[ea[t] * m + eb[t]] -= acc[t];
  __syncthreads();
  // in-place lower Cholesky (right-looking)
  for (int j = 0; j < m; ++j) {
    if (tid == 0) {
      const double v = sm.S[j * m + j];
      if (!(v > 0.0) || !isfinite(v)) sm.fail = 1;
      sm.S[j * m + j] = sqrt(v > 0.0 ? v : 1.0);
    }
    __syncthreads();
    const double djj = sm.S[j * m + j];
    for (int a = j + 1 + tid; a < m; a += FS_T) sm.S[a * m + j] /= djj;
    __syncthreads();
    const int rr = m - j - 1;
    for (int e = tid; e < rr * rr; e += FS_T) {
      const int a = j + 1 + e / rr, b = j + 1 + e % rr;
      if (b <= a) sm.S[a * m + b] -= sm.S[a * m + j] * sm.S[b * m + j];
    }
    __syncthreads();
  }
  // back-solve L^T z = e_{m-1} (one warp)
  if (tid < 32) {
    if (tid == 0) sm.z[m - 1] = 1.0 / sm.S[(m - 1) * m + (m - 1)];
    __syncwarp();
    for (int a = m - 2; a >= 0; --a) {
      double v = 0.0;
      for (int b = a + 1 + tid; b < m; b += 32) v = fma(sm.S[b * m + a], sm.z[b], v);
      v = warp_sum(v);
      if (tid == 0) sm.z[a] = -v / sm.S[a * m + a];
      __syncwarp();
    }
  }
  __syncthreads();
  const int npt1 = npt + 1;
  for (int t = tid; t < npt1; t += FS_T) {
    gval[(int64_t)t * n2 + i] = t < m ? sm.z[t] : 0.0;
    gcol[(int64_t)t * n2 + i] = t < m ? sm.idx[t] : -1;
  }
  if (tid == 0 && sm.fail) atomicMin(status, (int)i);
}

// ------------------------------------------------------------------ application kernels
// bp[c * n + r] = b[perm[r] * b_rs + c * b_cs]
__global__ void gather_rows_kernel(int64_t n, const int64_t* __restrict__ perm, const double* __restrict__ b,
                                   int64_t b_rs, int64_t b_cs, double* __restrict__ bp) {
  const int c = blockIdx.y;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    bp[(int64_t)c * n + r] = b[perm[r] * b_rs + c * b_cs];
}

// y[c * n2 + i] = sum_t G[i, t] x[c * n2 + col(i, t)]   (ELL, slot-major)
__global__ void ell_spmv_kernel(int64_t n2, int npt1, const double* __restrict__ gval,
                                const int32_t* __restrict__ gcol, const double* __restrict__ x,
                                double* __restrict__ y) {
  const int c = blockIdx.y;
  const double* xc = x + (int64_t)c * n2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int t = 0; t < npt1; ++t) {
      const int32_t j = gcol[(int64_t)t * n2 + i];
      if (j >= 0) v = fma(gval[(int64_t)t * n2 + i], xc[j], v);
    }
    y[(int64_t)c * n2 + i] = v;
  }
}

// u[c * n2 + j] = sum over rows i of column j of G: G[i, j] v[c * n2 + i]   (CSR of G^T, rows ascending)
__global__ void csr_spmv_kernel(int64_t n2, const int32_t* __restrict__ ptr, const int32_t* __restrict__ row,
                                const double* __restrict__ val, const double* __restrict__ v,
                                double* __restrict__ u) {
  const int c = blockIdx.y;
  const double* vc = v + (int64_t)c * n2;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n2; j += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int32_t e = ptr[j]; e < ptr[j + 1]; ++e) a = fma(val[e], vc[row[e]], a);
    u[(int64_t)c * n2 + j] = a;
  }
}

// out[perm[r]] = r < m ? o1[c * m + r] : u2[c * n2 + r - m]
__global__ void scatter_rows_kernel(int64_t n, int64_t m, const int64_t* __restrict__ perm,
                                    const double* __restrict__ o1, const double* __restrict__ u2,
                                    double* __restrict__ out, int64_t o_rs, int64_t o_cs) {
  const int c = blockIdx.y;
  const int64_t n2 = n - m;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const double v = r < m ? o1[(int64_t)c * m + r] : u2[(int64_t)c * n2 + (r - m)];
    out[perm[r] * o_rs + c * o_cs] = v;
  }
}

// ---- point-major variants (k > 8 right-hand sides): every block stored (rows x k) with the
// k values of a point contiguous, so the sparse products gather whole 8k-byte rows (one
// coalesced read per neighbour instead of k scattered ones) and the dense products are the
// transposed GEMMs (cuBLAS, column-major k x rows).
constexpr int PM_T = 32;  // transpose tile (rows x columns)

// bp[r * k + c] = b[perm[r] * b_rs + c * b_cs]   (tile transpose through shared memory)
__global__ void pm_gather_kernel(int64_t n, int64_t k, const int64_t* __restrict__ perm, const double* __restrict__ b,
                                 int64_t b_rs, int64_t b_cs, double* __restrict__ bp) {
  __shared__ double tile[PM_T][PM_T + 1];
  const int64_t r0 = (int64_t)blockIdx.x * PM_T, c0 = (int64_t)blockIdx.y * PM_T;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t r = r0 + tx;
  const int64_t pr = r < n ? perm[r] : 0;
  for (int cc = ty; cc < PM_T; cc += blockDim.y)
    if (r < n && c0 + cc < k) tile[cc][tx] = b[pr * b_rs + (c0 + cc) * b_cs];
  __syncthreads();
  for (int rr = ty; rr < PM_T; rr += blockDim.y)
    if (r0 + rr < n && c0 + tx < k) bp[(r0 + rr) * k + c0 + tx] = tile[tx][rr];
}

// out[perm[r] * o_rs + c * o_cs] = r < m ? o1[r * k + c] : u2[(r - m) * k + c]
__global__ void pm_scatter_kernel(int64_t n, int64_t m, int64_t k, const int64_t* __restrict__ perm,
                                  const double* __restrict__ o1, const double* __restrict__ u2,
                                  double* __restrict__ out, int64_t o_rs, int64_t o_cs) {
  __shared__ double tile[PM_T][PM_T + 1];
  const int64_t r0 = (int64_t)blockIdx.x * PM_T, c0 = (int64_t)blockIdx.y * PM_T;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int rr = ty; rr < PM_T; rr += blockDim.y) {
    const int64_t r = r0 + rr;
    if (r < n && c0 + tx < k) tile[tx][rr] = r < m ? o1[r * k + c0 + tx] : u2[(r - m) * k + c0 + tx];
  }
  __syncthreads();
  const int64_t r = r0 + tx;
  if (r >= n) return;
  const int64_t pr = perm[r];
  for (int cc = ty; cc < PM_T; cc += blockDim.y)
    if (c0 + cc < k) out[pr * o_rs + (c0 + cc) * o_cs] = tile[cc][tx];
}

// y[i * k + c] = sum_t G[i, t] x[col(i, t) * k + c]   (ELL, slot-major; thread = (i, c))
__global__ void pm_ell_kernel(int64_t n2, int64_t k, int npt1, const double* __restrict__ gval,
                              const int32_t* __restrict__ gcol, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n2 * k) return;
  const int64_t i = e / k, c = e - i * k;
  double v = 0.0;
  for (int t = 0; t < npt1; ++t) {
    const int32_t j = gcol[(int64_t)t * n2 + i];
    if (j >= 0) v = fma(gval[(int64_t)t * n2 + i], x[(int64_t)j * k + c], v);
  }
  y[e] = v;
}

// u[j * k + c] = sum over rows i of column j of G: G[i, j] v[i * k + c]   (CSR of G^T, rows ascending)
__global__ void pm_csr_kernel(int64_t n2, int64_t k, const int32_t* __restrict__ ptr, const int32_t* __restrict__ row,
                              const double* __restrict__ val, const double* __restrict__ v, double* __restrict__ u) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n2 * k) return;
  const int64_t j = e / k, c = e - j * k;
  double a = 0.0;
  for (int32_t q = ptr[j]; q < ptr[j + 1]; ++q) a = fma(val[q], v[(int64_t)row[q] * k + c], a);
  u[e] = a;
}

// ------------------------------------------------------------------ sampling z ~ N(0, M)
// level relaxation for the forward substitution G x = b: level(i) = 1 + max level of the
// earlier neighbours; Jacobi sweeps converge in (depth) sweeps (values only increase)
__global__ void afn_level_relax_kernel(int64_t n2, int npt1, const int32_t* __restrict__ gcol, int32_t* level,
                                       int32_t* changed) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  int l = 0;
  for (int t = 0; t < npt1; ++t) {
    const int32_t j = gcol[(int64_t)t * n2 + i];
    if (j >= 0 && j != i) {
      const int lj = ((volatile int32_t*)level)[j] + 1;
      l = lj > l ? lj : l;
    }
  }
  if (l > level[i]) {
    level[i] = l;
    *changed = 1;
  }
}

// one level of the forward substitution, every column: x_i = (b_i - sum_j G_ij x_j) / G_ii
__global__ void afn_level_solve_kernel(const int32_t* __restrict__ rows, int cnt, int64_t n2, int npt1,
                                       const double* __restrict__ gval, const int32_t* __restrict__ gcol,
                                       const double* __restrict__ b, double* __restrict__ x) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cnt) return;
  const int c = blockIdx.y;
  const int64_t i = rows[e];
  const double* xc = x + (int64_t)c * n2;
  double acc = b[(int64_t)c * n2 + i], diag = 1.0;
  // eight slots at a time: their index/value loads, then their x gathers, are issued
  // together (the one-slot loop was a chain of dependent load pairs: ~29 us per level at
  // n2 = 64512); accumulation order stays t ascending
  for (int t0 = 0; t0 < npt1; t0 += 8) {
    int32_t j[8];
    double g[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u;
      j[u] = t < npt1 ? gcol[(int64_t)t * n2 + i] : -1;
      g[u] = t < npt1 ? gval[(int64_t)t * n2 + i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = (j[u] >= 0 && j[u] != i) ? xc[j[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j[u] < 0) continue;
      if (j[u] == i)
        diag = g[u];
      else
        acc = fma(-g[u], xv[u], acc);
    }
  }
  x[(int64_t)c * n2 + i] = acc / diag;
}

// z[c*n + perm[r]] = r < m ? z1[c*m + r] : t[c*n2 + r - m] + x[c*n2 + r - m]
__global__ void afn_assemble_kernel(int64_t n, int64_t m, const int64_t* __restrict__ perm,
                                    const double* __restrict__ z1, const double* __restrict__ t,
                                    const double* __restrict__ x, double* __restrict__ z) {
  const int c = blockIdx.y;
  const int64_t n2 = n - m;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const double v = r < m ? z1[(int64_t)c * m + r] : t[(int64_t)c * n2 + r - m] + x[(int64_t)c * n2 + r - m];
    z[(int64_t)c * n + perm[r]] = v;
  }
}

// b[c*n2 + i] = w[(m + i) * w_rs + c * w_cs]
__global__ void afn_gather_tail_kernel(int64_t n2, int64_t m, const double* __restrict__ w, int64_t w_rs,
                                       int64_t w_cs, double* __restrict__ b) {
  const int c = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
    b[(int64_t)c * n2 + i] = w[(m + i) * w_rs + c * w_cs];
}

// ------------------------------------------------------------------ local predictive variance
// var(x*) ~= f^2 - c^T (Khat_NN)^-1 c over the K nearest training points N of x* (local
// kriging): one CTA per test point, S_NN = f^2 kappa + s I and c = f^2 kappa(x*, x_N) in
// shared memory, Cholesky, var = f^2 - |L^-1 c|^2.
constexpr int LV_MAXM = KNN_MAX_CROSS;  // 128 x 128 fp64 block: 128 KB of shared memory
struct LvSmem {
  double S[LV_MAXM * LV_MAXM];
  double xs[LV_MAXM * 16];
  double c[LV_MAXM];
  double q[16];
  int idx[LV_MAXM];
  int m;
  int fail;
};

template <int KT>
__global__ void __launch_bounds__(FS_T) local_var_kernel(int64_t nq, int d, const double* __restrict__ xq,
                                                         const double* __restrict__ x, double l, double f2, double s,
                                                         int npt, const int64_t* __restrict__ nbr,
                                                         double* __restrict__ var, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LvSmem& sm = *reinterpret_cast<LvSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int64_t i = blockIdx.x;
  if (tid == 0) {
    int m = 0;
    for (int t = 0; t < npt; ++t) {
      const int64_t j = nbr[i * npt + t];
      if (j >= 0) sm.idx[m++] = (int)j;
    }
    sm.m = m;
    sm.fail = 0;
  }
  if (tid < d) sm.q[tid] = xq[i * d + tid];
  __syncthreads();
  const int m = sm.m;
  for (int e = tid; e < m * d; e += FS_T) sm.xs[e] = x[(int64_t)sm.idx[e / d] * d + e % d];
  __syncthreads();
  for (int e = tid; e < m * m + m; e += FS_T) {
    double r2 = 0.0;
    if (e < m * m) {
      const int a = e / m, b = e % m;
      if (b > a) continue;
      for (int c = 0; c < d; ++c) {
        const double df = sm.xs[a * d + c] - sm.xs[b * d + c];
        r2 = fma(df, df, r2);
      }
      sm.S[a * m + b] = f2 * kappa64<KT>(r2, l) + (a == b ? s : 0.0);
    } else {
      const int a = e - m * m;
      for (int c = 0; c < d; ++c) {
        const double df = sm.xs[a * d + c] - sm.q[c];
        r2 = fma(df, df, r2);
      }
      sm.c[a] = f2 * kappa64<KT>(r2, l);
    }
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {  // in-place lower Cholesky
    if (tid == 0) {
      const double v = sm.S[j * m + j];
      if (!(v > 0.0) || !isfinite(v)) sm.fail = 1;
      sm.S[j * m + j] = sqrt(v > 0.0 ? v : 1.0);
    }
    __syncthreads();
    const double djj = sm.S[j * m + j];
    for (int a = j + 1 + tid; a < m; a += FS_T) sm.S[a * m + j] /= djj;
    __syncthreads();
    const int rr = m - j - 1;
    for (int e = tid; e < rr * rr; e += FS_T) {
      const int a = j + 1 + e / rr, b = j + 1 + e % rr;
      if (b <= a) sm.S[a * m + b] -= sm.S[a * m + j] * sm.S[b * m + j];
    }
    __syncthreads();
  }
  if (tid < 32) {  // forward solve L y = c (in place in c), var = f^2 - |y|^2
    for (int a = 0; a < m; ++a) {
      double v = 0.0;
      for (int b = tid; b < a; b += 32) v = fma(sm.S[a * m + b], sm.c[b], v);
      v = warp_sum(v);
      if (tid == 0) sm.c[a] = (sm.c[a] - v) / sm.S[a * m + a];
      __syncwarp();
    }
    double ss = 0.0;
    for (int a = tid; a < m; a += 32) ss = fma(sm.c[a], sm.c[a], ss);
    ss = warp_sum(ss);
    if (tid == 0) {
      const double v = f2 - ss;
      var[i] = v > 0.0 ? v : 0.0;
      if (sm.fail) atomicMin(status, (int)i);
    }
  }
}

inline dim3 vec_grid(int64_t n, int64_t k) {
  int64_t bx = (n + 255) / 256;
  if (bx > 592) bx = 592;
  return dim3((unsigned)(bx > 0 ? bx : 1), (unsigned)k);
}

}  // namespace

// M^-1 B for k > 8 right-hand sides in the point-major layout (same algebra as below).
static int afn_apply_pm(kgp_precond_s* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* out,
                        int64_t o_rs, int64_t o_cs, cudaStream_t st) {
  const int64_t n = p->n, m = p->m, n2 = p->n2;
  int rc = p->work.ensure(sizeof(double) * (size_t)k * (n + 3 * n2 + 3 * m));
  if (rc) return rc;
  double* bp = p->work.as<double>();  // (n x k): rows [0, m) = b1, [m, n) = b2
  double* y1 = bp + k * n;
  double* t2 = y1 + k * m;
  double* v = t2 + k * n2;
  double* u2 = v + k * n2;
  double* z1 = u2 + k * n2;
  double* o1 = z1 + k * m;
  const int64_t* perm = p->perm.as<int64_t>();
  const double* linv = p->linv.as<double>();
  const double* w = p->w.as<double>();
  const dim3 tgrid((unsigned)((n + PM_T - 1) / PM_T), (unsigned)((k + PM_T - 1) / PM_T));
  pm_gather_kernel<<<tgrid, dim3(PM_T, 8), 0, st>>>(n, k, perm, b, b_rs, b_cs, bp);
  KGP_LAUNCH("pm_gather_kernel");
  // transposed products, C^T (k x rows, column-major) = B^T A^T:
  // y1 = L^-1 b1
  rc = gemm_f64(k, m, m, bp, 1, k, linv, 1, m, y1, 1, k, 1.0, 0.0, nullptr, 0, 0, p->tmp, st);
  if (rc) return rc;
  // W products: the DMMA streams of wgemm.cu where they beat cuBLAS DGEMM -- 33..40 columns,
  // which a 32-wide library tile pads to 64; env KGP_AFN_WGEMM=0 never,
  // =2 for every k <= 64 (tests, measurements)
  const char* wge = getenv("KGP_AFN_WGEMM");
  const int wg_mode = wge ? atoi(wge) : 1;
  const bool wg = wg_mode != 0 && wgemm_supported(m, k, w, m) && (wg_mode == 2 || (k >= 33 && k <= 40));
  // t2 = b2 - W y1
  rc = wg ? wy_product(n2, m, k, w, m, y1, k, 1, t2, k, 1, -1.0, 1.0, bp + m * k, k, 1, st)
          : gemm_f64(k, n2, m, y1, 1, k, w, 1, m, t2, 1, k, -1.0, 1.0, bp + m * k, 1, k, p->tmp, st);
  if (rc) return rc;
  // u2 = G^T (G t2)
  const unsigned sgrid = (unsigned)((n2 * k + 255) / 256);
  pm_ell_kernel<<<sgrid, 256, 0, st>>>(n2, k, p->npt1, p->gval.as<double>(), p->gcol.as<int32_t>(), t2, v);
  KGP_LAUNCH("pm_ell_kernel");
  pm_csr_kernel<<<sgrid, 256, 0, st>>>(n2, k, p->gtptr.as<int32_t>(), p->gtrow.as<int32_t>(), p->gtval.as<double>(),
                                       v, u2);
  KGP_LAUNCH("pm_csr_kernel");
  // z1 = y1 - W^T u2
  rc = wg ? wtu_product(n2, m, k, w, m, u2, k, 1, z1, k, 1, -1.0, 1.0, y1, k, 1, p->tmp, st)
          : gemm_f64(k, m, n2, u2, 1, k, w, m, 1, z1, 1, k, -1.0, 1.0, y1, 1, k, p->tmp, st);
  if (rc) return rc;
  // o1 = L^-T z1
  rc = gemm_f64(k, m, m, z1, 1, k, linv, m, 1, o1, 1, k, 1.0, 0.0, nullptr, 0, 0, p->tmp, st);
  if (rc) return rc;
  pm_scatter_kernel<<<tgrid, dim3(PM_T, 8), 0, st>>>(n, m, k, perm, o1, u2, out, o_rs, o_cs);
  KGP_LAUNCH("pm_scatter_kernel");
  return KGP_OK;
}

int afn_apply_impl(kgp_precond_s* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* out,
                   int64_t o_rs, int64_t o_cs, cudaStream_t st) {
  KGP_REQUIRE(k <= 65535, KGP_ERR_INVALID, "too many right-hand sides (%lld)", (long long)k);
  static const bool pm = [] {
    const char* e = getenv("KGP_AFN_PM");
    return !(e && atoi(e) == 0);
  }();
  if (pm && k > 8) return afn_apply_pm(p, k, b, b_rs, b_cs, out, o_rs, o_cs, st);
  const int64_t n = p->n, m = p->m, n2 = p->n2;
  // workspace (column-major blocks): bp (n), y1 (m), t2 (n2), v (n2), u2 (n2), z1 (m), o1 (m)
  int rc = p->work.ensure(sizeof(double) * (size_t)k * (n + 3 * n2 + 3 * m));
  if (rc) return rc;
  double* bp = p->work.as<double>();
  double* y1 = bp + k * n;
  double* t2 = y1 + k * m;
  double* v = t2 + k * n2;
  double* u2 = v + k * n2;
  double* z1 = u2 + k * n2;
  double* o1 = z1 + k * m;
  const int64_t* perm = p->perm.as<int64_t>();
  const double* linv = p->linv.as<double>();
  const double* w = p->w.as<double>();
  gather_rows_kernel<<<vec_grid(n, k), 256, 0, st>>>(n, perm, b, b_rs, b_cs, bp);
  KGP_LAUNCH("gather_rows_kernel");
  // y1 = L^-1 b1
  rc = gemm_f64(m, k, m, linv, m, 1, bp, 1, n, y1, 1, m, 1.0, 0.0, nullptr, 0, 0, p->tmp, st);
  if (rc) return rc;
  // t2 = b2 - W y1
  rc = gemm_f64(n2, k, m, w, m, 1, y1, 1, m, t2, 1, n2, -1.0, 1.0, bp + m, 1, n, p->tmp, st);
  if (rc) return rc;
  // u2 = G^T (G t2)
  ell_spmv_kernel<<<vec_grid(n2, k), 256, 0, st>>>(n2, p->npt1, p->gval.as<double>(), p->gcol.as<int32_t>(), t2, v);
  KGP_LAUNCH("ell_spmv_kernel");
  csr_spmv_kernel<<<vec_grid(n2, k), 256, 0, st>>>(n2, p->gtptr.as<int32_t>(), p->gtrow.as<int32_t>(),
                                                   p->gtval.as<double>(), v, u2);
  KGP_LAUNCH("csr_spmv_kernel");
  // z1 = y1 - W^T u2
  rc = gemm_f64(m, k, n2, w, 1, m, u2, 1, n2, z1, 1, m, -1.0, 1.0, y1, 1, m, p->tmp, st);
  if (rc) return rc;
  // o1 = L^-T z1
  rc = gemm_f64(m, k, m, linv, 1, m, z1, 1, m, o1, 1, m, 1.0, 0.0, nullptr, 0, 0, p->tmp, st);
  if (rc) return rc;
  scatter_rows_kernel<<<vec_grid(n, k), 256, 0, st>>>(n, m, perm, o1, u2, out, o_rs, o_cs);
  KGP_LAUNCH("scatter_rows_kernel");
  return KGP_OK;
}

// rows of the FSAI factor grouped by dependency level (computed once per handle)
static int afn_levels(kgp_precond_s* p, cudaStream_t st) {
  if (!p->lvl_ptr.empty()) return KGP_OK;
  const int64_t n2 = p->n2;
  DevBuf lv;
  int rc = lv.ensure(sizeof(int32_t) * (n2 + 1));
  if (rc) return rc;
  int32_t* level = lv.as<int32_t>();
  int32_t* changed = level + n2;
  KGP_CUDA(cudaMemsetAsync(level, 0, sizeof(int32_t) * (n2 + 1), st));
  for (int it = 0;; ++it) {
    KGP_REQUIRE(it <= n2 + 1, KGP_ERR_NUMERICAL, "FSAI dependency levels did not converge");
    int32_t h = 0;
    KGP_CUDA(cudaMemsetAsync(changed, 0, sizeof(int32_t), st));
    afn_level_relax_kernel<<<(unsigned)((n2 + 255) / 256), 256, 0, st>>>(n2, p->npt1, p->gcol.as<int32_t>(), level,
                                                                        changed);
    KGP_LAUNCH("afn_level_relax_kernel");
    KGP_CUDA(cudaMemcpyAsync(&h, changed, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KGP_CUDA(cudaStreamSynchronize(st));
    if (!h) break;
  }
  std::vector<int32_t> hl(n2);
  KGP_CUDA(cudaMemcpy(hl.data(), level, sizeof(int32_t) * n2, cudaMemcpyDeviceToHost));
  int32_t depth = 0;
  for (int32_t v : hl) depth = v + 1 > depth ? v + 1 : depth;
  std::vector<int64_t> ptr(depth + 1, 0);
  for (int32_t v : hl) ++ptr[v + 1];
  for (int32_t L = 0; L < depth; ++L) ptr[L + 1] += ptr[L];
  std::vector<int32_t> rows(n2);
  std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
  for (int64_t i = 0; i < n2; ++i) rows[pos[hl[i]]++] = (int32_t)i;  // ascending rows within a level
  rc = p->lvl_rows.ensure(sizeof(int32_t) * n2);
  if (rc) return rc;
  KGP_CUDA(cudaMemcpy(p->lvl_rows.p, rows.data(), sizeof(int32_t) * n2, cudaMemcpyHostToDevice));
  p->lvl_ptr = ptr;
  return KGP_OK;
}

}  // namespace kgp

using namespace kgp;

extern "C" int kgp_afn_sample(kgp_precond* p, int64_t k, const double* w, int64_t w_rs, int64_t w_cs, double* z,
                              void* stream) {
  KGP_REQUIRE(p != nullptr && p->magic == PRECOND_MAGIC && p->kind == KGP_PRECOND_AFN, KGP_ERR_STATE,
              "kgp_afn_sample needs an AFN handle");
  KGP_REQUIRE(p->l11.p != nullptr, KGP_ERR_INVALID, "this AFN handle was created without its landmark factor");
  KGP_REQUIRE(k >= 1 && k <= 65535 && w != nullptr && z != nullptr, KGP_ERR_INVALID, "bad sample arguments");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = afn_levels(p, st);
  if (rc) return rc;
  const int64_t n = p->n, m = p->m, n2 = p->n2;
  rc = p->swork.ensure(sizeof(double) * (size_t)k * (m + 3 * n2));
  if (rc) return rc;
  double* z1 = p->swork.as<double>();
  double* t = z1 + k * m;
  double* b = t + k * n2;
  double* x = b + k * n2;
  // z1 = L11 w1;  t = W w1  (w1: rows 0..m-1 of w)
  rc = gemm_f64(m, k, m, p->l11.as<double>(), m, 1, w, w_rs, w_cs, z1, 1, m, 1.0, 0.0, nullptr, 0, 0, p->tmp, st);
  if (rc) return rc;
  rc = gemm_f64(n2, k, m, p->w.as<double>(), m, 1, w, w_rs, w_cs, t, 1, n2, 1.0, 0.0, nullptr, 0, 0, p->tmp, st);
  if (rc) return rc;
  // x = G^-1 w2, level by level
  afn_gather_tail_kernel<<<vec_grid(n2, k), 256, 0, st>>>(n2, m, w, w_rs, w_cs, b);
  KGP_LAUNCH("afn_gather_tail_kernel");
  const int32_t* rows = p->lvl_rows.as<int32_t>();
  for (size_t L = 0; L + 1 < p->lvl_ptr.size(); ++L) {
    const int64_t r0 = p->lvl_ptr[L], cnt = p->lvl_ptr[L + 1] - r0;
    afn_level_solve_kernel<<<dim3((unsigned)((cnt + 127) / 128), (unsigned)k), 128, 0, st>>>(
        rows + r0, (int)cnt, n2, p->npt1, p->gval.as<double>(), p->gcol.as<int32_t>(), b, x);
    KGP_LAUNCH("afn_level_solve_kernel");
  }
  afn_assemble_kernel<<<vec_grid(n, k), 256, 0, st>>>(n, m, p->perm.as<int64_t>(), z1, t, x, z);
  KGP_LAUNCH("afn_assemble_kernel");
  return KGP_OK;
}

extern "C" int kgp_knn_prev(int64_t n, int d, const double* x, int npt, int64_t* idx_out, void* stream) {
  KGP_REQUIRE(n >= 0 && d >= 1 && d <= 16, KGP_ERR_INVALID, "dimension d=%d outside [1, 16]", d);
  KGP_REQUIRE(npt >= 1 && npt <= KNN_MAX, KGP_ERR_INVALID, "npt=%d outside [1, %d]", npt, KNN_MAX);
  KGP_REQUIRE(n == 0 || (x != nullptr && idx_out != nullptr), KGP_ERR_INVALID, "NULL pointer");
  if (n == 0) return KGP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = (unsigned)((n + KNN_T - 1) / KNN_T);
  switch (d) {
#define KGP_KNN_CASE(D)                                                \
  case D:                                                              \
    knn_kernel<D, true><<<grid, KNN_T, 0, st>>>(n, x, n, x, npt, idx_out); \
    break;
    KGP_KNN_CASE(1) KGP_KNN_CASE(2) KGP_KNN_CASE(3) KGP_KNN_CASE(4) KGP_KNN_CASE(5) KGP_KNN_CASE(6)
    KGP_KNN_CASE(7) KGP_KNN_CASE(8) KGP_KNN_CASE(9) KGP_KNN_CASE(10) KGP_KNN_CASE(11) KGP_KNN_CASE(12)
    KGP_KNN_CASE(13) KGP_KNN_CASE(14) KGP_KNN_CASE(15) KGP_KNN_CASE(16)
#undef KGP_KNN_CASE
  }
  KGP_LAUNCH("knn_kernel");
  return KGP_OK;
}

extern "C" int kgp_knn_cross(int64_t nq, const double* xq, int64_t nx, const double* x, int d, int npt,
                             int64_t* idx_out, void* stream) {
  KGP_REQUIRE(nq >= 0 && nx >= 1 && d >= 1 && d <= 16, KGP_ERR_INVALID, "bad kNN shapes (d=%d)", d);
  KGP_REQUIRE(npt >= 1 && npt <= KNN_MAX_CROSS, KGP_ERR_INVALID, "npt=%d outside [1, %d]", npt, KNN_MAX_CROSS);
  KGP_REQUIRE(nq == 0 || (xq != nullptr && x != nullptr && idx_out != nullptr), KGP_ERR_INVALID, "NULL pointer");
  if (nq == 0) return KGP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = (unsigned)((nq + KNN_T - 1) / KNN_T);
  switch (d) {
#define KGP_KNNX_CASE(D)                                                        \
  case D:                                                                       \
    if (npt <= KNN_MAX)                                                         \
      knn_kernel<D, false><<<grid, KNN_T, 0, st>>>(nq, xq, nx, x, npt, idx_out); \
    else                                                                        \
      knn_kernel<D, false, KNN_MAX_CROSS><<<grid, KNN_T, 0, st>>>(nq, xq, nx, x, npt, idx_out); \
    break;
    KGP_KNNX_CASE(1) KGP_KNNX_CASE(2) KGP_KNNX_CASE(3) KGP_KNNX_CASE(4) KGP_KNNX_CASE(5) KGP_KNNX_CASE(6)
    KGP_KNNX_CASE(7) KGP_KNNX_CASE(8) KGP_KNNX_CASE(9) KGP_KNNX_CASE(10) KGP_KNNX_CASE(11) KGP_KNNX_CASE(12)
    KGP_KNNX_CASE(13) KGP_KNNX_CASE(14) KGP_KNNX_CASE(15) KGP_KNNX_CASE(16)
#undef KGP_KNNX_CASE
  }
  KGP_LAUNCH("knn_kernel");
  return KGP_OK;
}

extern "C" int kgp_local_variance(int kernel, int64_t nq, int d, const double* xq, const double* x, double l,
                                  double f, double s, int npt, const int64_t* nbr, double* var, void* stream) {
  KGP_REQUIRE(kernel >= 0 && kernel <= 2, KGP_ERR_INVALID, "unknown kernel id %d", kernel);
  KGP_REQUIRE(d >= 1 && d <= 16 && npt >= 1 && npt <= KNN_MAX_CROSS && nq >= 0 && nq < ((int64_t)1 << 31),
              KGP_ERR_INVALID, "bad local-variance shapes (npt <= %d)", KNN_MAX_CROSS);
  KGP_REQUIRE(l > 0.0 && s > 0.0, KGP_ERR_INVALID, "length scale and noise must be positive");
  if (nq == 0) return KGP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf status;
  int rc = status.ensure(sizeof(int32_t));
  if (rc) return rc;
  KGP_CUDA(cudaMemsetAsync(status.p, 0x7f, sizeof(int32_t), st));
  const size_t smem = sizeof(LvSmem);
  switch (kernel) {
#define KGP_LV_CASE(K)                                                                                          \
  case K: {                                                                                                     \
    KGP_SMEM_ATTR(local_var_kernel<K>, smem);                                                            \
    local_var_kernel<K><<<(unsigned)nq, FS_T, smem, st>>>(nq, d, xq, x, l, f * f, s, npt, nbr, var,            \
                                                          status.as<int32_t>());                                \
    break;                                                                                                      \
  }
    KGP_LV_CASE(0) KGP_LV_CASE(1) KGP_LV_CASE(2)
#undef KGP_LV_CASE
  }
  KGP_LAUNCH("local_var_kernel");
  int32_t bad = 0;
  KGP_CUDA(cudaMemcpyAsync(&bad, status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  KGP_CUDA(cudaStreamSynchronize(st));
  KGP_REQUIRE(bad == 0x7f7f7f7f, KGP_ERR_NUMERICAL, "local covariance block of test point %d is not SPD", bad);
  return KGP_OK;
}

extern "C" int kgp_afn_fsai(int kernel, int64_t n2, int d, const double* x2, double l, double f, double s,
                            const double* dshift, int64_t m, const double* w, int npt, const int64_t* nbr,
                            double* gval, int32_t* gcol, void* stream) {
  KGP_REQUIRE(kernel >= 0 && kernel <= 2, KGP_ERR_INVALID, "unknown kernel id %d", kernel);
  KGP_REQUIRE(d >= 1 && d <= 16, KGP_ERR_INVALID, "dimension d=%d outside [1, 16]", d);
  KGP_REQUIRE(npt >= 1 && npt <= KNN_MAX, KGP_ERR_INVALID, "npt=%d outside [1, %d]", npt, KNN_MAX);
  KGP_REQUIRE(n2 >= 1 && n2 < (int64_t)1 << 31 && m >= 0, KGP_ERR_INVALID, "bad sizes n2=%lld m=%lld",
              (long long)n2, (long long)m);
  KGP_REQUIRE(l > 0.0 && s > 0.0, KGP_ERR_INVALID, "length scale and noise must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf status;
  int rc = status.ensure(sizeof(int32_t));
  if (rc) return rc;
  KGP_CUDA(cudaMemsetAsync(status.p, 0x7f, sizeof(int32_t), st));
  const size_t smem = sizeof(FsaiSmem);
  const double f2 = f * f;
  switch (kernel) {
#define KGP_FSAI_CASE(K)                                                                                   \
  case K: {                                                                                                \
    KGP_SMEM_ATTR(fsai_kernel<K>, smem);                                                            \
    fsai_kernel<K><<<(unsigned)n2, FS_T, smem, st>>>(n2, d, x2, l, f2, s, m, w, npt, nbr, dshift, gval,    \
                                                    gcol, status.as<int32_t>());                           \
    break;                                                                                                 \
  }
    KGP_FSAI_CASE(0) KGP_FSAI_CASE(1) KGP_FSAI_CASE(2)
#undef KGP_FSAI_CASE
  }
  KGP_LAUNCH("fsai_kernel");
  int32_t bad = 0;
  KGP_CUDA(cudaMemcpyAsync(&bad, status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  KGP_CUDA(cudaStreamSynchronize(st));
  KGP_REQUIRE(bad == 0x7f7f7f7f, KGP_ERR_BREAKDOWN,
              "FSAI block of row %d is not positive definite (Schur complement lost definiteness)", bad);
  return KGP_OK;
}
