// Fused kernel-matrix MatMul in fp64 (precision KGP_FP64): the parity anchor.
//
// Same contract as KernelEngine._streamed_matmul (kmat.py:165-189): per entry a
// direct-difference r^2 in fp64 (_panels_numba.py:23-34 order), the kernel and
// its l-derivative (_panels_numba.py:37-131), contracted against the RHS block
// in fp64. The tile lives in shared memory only; Khat is never stored.
// CTA = 64 rows x (up to) 64 RHS columns, 128 threads, 16-column j tiles.
#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

constexpr int TR = 64;   // rows per CTA
constexpr int TJ = 16;   // columns per j tile (static smem stays < 48 KB)
constexpr int NT = 128;  // threads
constexpr int MAXD = 16;

template <int KT, int NOUT, int CT>
__global__ void __launch_bounds__(NT) kmm_f64_kernel(const F64Params p) {
  const int kp = CT * 8;
  __shared__ double sXr[TR][MAXD + 1];
  __shared__ double sXj[TJ][MAXD + 1];
  __shared__ double sK[TR][TJ + 1];
  __shared__ double sG[NOUT == 2 ? TR : 1][TJ + 1];
  __shared__ double sB[TJ][64];

  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * TR;
  const int c0 = blockIdx.y * 64;  // RHS slice
  const int d = p.d;

  for (int e = tid; e < TR * d; e += NT) {
    int r = e / d, q = e % d;
    sXr[r][q] = (row0 + r < p.nrows) ? p.xr[(row0 + r) * d + q] : 0.0;
  }
  const int rg = tid >> 3, cg = tid & 7;
  double acc[4][CT], accg[NOUT == 2 ? 4 : 1][CT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < CT; ++q) {
      acc[i][q] = 0.0;
      if (NOUT == 2) accg[i][q] = 0.0;
    }

  for (int64_t j0 = 0; j0 < p.ncols; j0 += TJ) {
    __syncthreads();
    for (int e = tid; e < TJ * d; e += NT) {
      int jj = e / d, q = e % d;
      sXj[jj][q] = (j0 + jj < p.ncols) ? p.xc[(j0 + jj) * d + q] : 0.0;
    }
    for (int e = tid; e < TJ * kp; e += NT) {
      int jj = e / kp, c = e % kp;
      int64_t j = j0 + jj;
      int cc = c0 + c;
      sB[jj][c] = (j < p.ncols && cc < p.k) ? p.b[j * p.b_rs + (int64_t)cc * p.b_cs] : 0.0;
    }
    __syncthreads();
    // tile: entries (r, jj), consecutive threads on consecutive columns
    for (int e = tid; e < TR * TJ; e += NT) {
      int r = e / TJ, jj = e % TJ;
      double r2 = 0.0;
      for (int q = 0; q < d; ++q) {
        double df = sXr[r][q] - sXj[jj][q];
        r2 = __dadd_rn(r2, __dmul_rn(df, df));  // numba's rounding (no FMA contraction)
      }
      bool valid = (j0 + jj) < p.ncols;
      sK[r][jj] = valid ? kappa64<KT>(r2, p.l) : 0.0;
      if (NOUT == 2) sG[r][jj] = valid ? dkappa64<KT>(r2, p.l) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int jj = 0; jj < TJ; ++jj) {
      double kv[4], gv[4], bv[CT];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        kv[i] = sK[rg * 4 + i][jj];
        if (NOUT == 2) gv[i] = sG[rg * 4 + i][jj];
      }
#pragma unroll
      for (int q = 0; q < CT; ++q) bv[q] = sB[jj][cg + 8 * q];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < CT; ++q) {
          acc[i][q] = fma(kv[i], bv[q], acc[i][q]);
          if (NOUT == 2) accg[i][q] = fma(gv[i], bv[q], accg[i][q]);
        }
    }
  }
  // epilogue (kmat.py:186-188): scale, + s B on the diagonal rows
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t r = row0 + rg * 4 + i;
    if (r >= p.nrows) continue;
#pragma unroll
    for (int q = 0; q < CT; ++q) {
      int c = c0 + cg + 8 * q;
      if (c >= p.k) continue;
      int64_t o = r * p.o_rs + (int64_t)c * p.o_cs;
      if (p.out_k) {
        double v = p.f2 * acc[i][q];
        if (p.diag_row0 >= 0) v += p.s * p.b[(p.diag_row0 + r) * p.b_rs + (int64_t)c * p.b_cs];
        p.out_k[o] = v;
      }
      if (p.out_df) p.out_df[o] = p.two_f * acc[i][q];
      if (NOUT == 2 && p.out_dl) p.out_dl[o] = p.f2_dl * accg[i][q];
    }
  }
}

template <int KT, int NOUT>
int launch_nout(const F64Params& p, cudaStream_t st) {
  int kslice = p.k < 64 ? p.k : 64;
  dim3 grid((unsigned)((p.nrows + TR - 1) / TR), (unsigned)((p.k + 63) / 64));
  if (kslice <= 8)
    kmm_f64_kernel<KT, NOUT, 1><<<grid, NT, 0, st>>>(p);
  else if (kslice <= 16)
    kmm_f64_kernel<KT, NOUT, 2><<<grid, NT, 0, st>>>(p);
  else if (kslice <= 32)
    kmm_f64_kernel<KT, NOUT, 4><<<grid, NT, 0, st>>>(p);
  else
    kmm_f64_kernel<KT, NOUT, 8><<<grid, NT, 0, st>>>(p);
  KGP_LAUNCH("kmm_f64_kernel");
  return KGP_OK;
}

template <int KT>
int launch_kt(const F64Params& p, cudaStream_t st) {
  return p.out_dl ? launch_nout<KT, 2>(p, st) : launch_nout<KT, 1>(p, st);
}

}  // namespace

int launch_kmm_f64(int kt, const F64Params& p, cudaStream_t st) {
  KGP_REQUIRE(p.d >= 1 && p.d <= MAXD, KGP_ERR_INVALID, "fp64 operator supports 1 <= d <= %d, got %d", MAXD, p.d);
  if (p.nrows <= 0) return KGP_OK;
  switch (kt) {
    case GAUSS: return launch_kt<GAUSS>(p, st);
    case MAT32: return launch_kt<MAT32>(p, st);
    case MAT52: return launch_kt<MAT52>(p, st);
  }
  set_error(KGP_ERR_INVALID, "unknown kernel id %d", kt);
  return KGP_ERR_INVALID;
}

}  // namespace kgp
