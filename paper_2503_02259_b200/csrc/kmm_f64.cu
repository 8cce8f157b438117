// Fused kernel-matrix MatMul in fp64 (precision KGP_FP64): the parity anchor.
//
// Same contract as KernelEngine._streamed_matmul (kmat.py:165-189): per entry a
// direct-difference r^2 in fp64 (_panels_numba.py:23-34 order, no FMA
// contraction), the kernel and its l-derivative (_panels_numba.py:37-131),
// contracted against the RHS block in fp64. The tile lives in shared memory
// only; Khat is never stored.
//
// CTA = 64 rows x (up to) 64 RHS columns, 128 threads, 16-column j tiles. When
// the row blocks alone cannot fill the GPU (configs[0]: n = 4096 -> 64 row
// blocks), the column range is split over grid.z and the partial sums are
// reduced in a fixed order by a second kernel (deterministic, no atomics).
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
  const int64_t jb = (int64_t)blockIdx.z * p.jchunk;
  const int64_t je = jb + p.jchunk < p.ncols ? jb + p.jchunk : p.ncols;

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

  for (int64_t j0 = jb; j0 < je; j0 += TJ) {
    __syncthreads();
    for (int e = tid; e < TJ * d; e += NT) {
      int jj = e / d, q = e % d;
      sXj[jj][q] = (j0 + jj < je) ? p.xc[(j0 + jj) * d + q] : 0.0;
    }
    for (int e = tid; e < TJ * kp; e += NT) {
      int jj = e / kp, c = e % kp;
      int64_t j = j0 + jj;
      int cc = c0 + c;
      sB[jj][c] = (j < je && cc < p.k) ? p.b[j * p.b_rs + (int64_t)cc * p.b_cs] : 0.0;
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
      bool valid = (j0 + jj) < je;
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
  // epilogue (kmat.py:186-188): scale, + s B on the diagonal rows; raw partials when split
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t r = row0 + rg * 4 + i;
    if (r >= p.nrows) continue;
#pragma unroll
    for (int q = 0; q < CT; ++q) {
      int c = c0 + cg + 8 * q;
      if (c >= p.k) continue;
      if (p.part) {
        const int64_t slot = ((int64_t)blockIdx.z * p.nrows + r) * p.k + c;
        p.part[slot] = acc[i][q];
        if (NOUT == 2) p.part[p.part_stride + slot] = accg[i][q];
        continue;
      }
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

// sum the column-split partials in split order, then the epilogue
__global__ void f64_reduce_kernel(const F64Params p, int nsplit) {
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

template <int KT, int NOUT>
int launch_nout(const F64Params& p, dim3 grid, cudaStream_t st) {
  int kslice = p.k < 64 ? p.k : 64;
  // RHS slice padded to a multiple of 8 (k = 1 + k_z = 17 runs 24 columns, not 32)
  if (kslice <= 8)
    kmm_f64_kernel<KT, NOUT, 1><<<grid, NT, 0, st>>>(p);
  else if (kslice <= 16)
    kmm_f64_kernel<KT, NOUT, 2><<<grid, NT, 0, st>>>(p);
  else if (kslice <= 24)
    kmm_f64_kernel<KT, NOUT, 3><<<grid, NT, 0, st>>>(p);
  else if (kslice <= 32)
    kmm_f64_kernel<KT, NOUT, 4><<<grid, NT, 0, st>>>(p);
  else if (kslice <= 48)
    kmm_f64_kernel<KT, NOUT, 6><<<grid, NT, 0, st>>>(p);
  else
    kmm_f64_kernel<KT, NOUT, 8><<<grid, NT, 0, st>>>(p);
  KGP_LAUNCH("kmm_f64_kernel");
  return KGP_OK;
}

template <int KT>
int launch_kt(const F64Params& p, dim3 grid, cudaStream_t st) {
  return p.out_dl ? launch_nout<KT, 2>(p, grid, st) : launch_nout<KT, 1>(p, grid, st);
}

}  // namespace

int launch_kmm_f64(int kt, const F64Params& p_in, DevBuf& ws, cudaStream_t st) {
  KGP_REQUIRE(p_in.d >= 1 && p_in.d <= MAXD, KGP_ERR_INVALID, "fp64 operator supports 1 <= d <= %d, got %d", MAXD,
              p_in.d);
  KGP_REQUIRE(kt >= 0 && kt <= 2, KGP_ERR_INVALID, "unknown kernel id %d", kt);
  if (p_in.nrows <= 0) return KGP_OK;
  F64Params p = p_in;
  const int64_t rblk = (p.nrows + TR - 1) / TR, kslc = (p.k + 63) / 64;
  // split the columns until ~8 CTAs per SM are in flight (148 SMs), at >= 256 columns per split
  int64_t nsplit = (8 * 148 + rblk * kslc - 1) / (rblk * kslc);
  const int64_t maxsplit = p.ncols / 256 > 0 ? p.ncols / 256 : 1;
  if (nsplit > maxsplit) nsplit = maxsplit;
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
  int rc = (kt == GAUSS) ? launch_kt<GAUSS>(p, grid, st) : (kt == MAT32) ? launch_kt<MAT32>(p, grid, st)
                                                                            : launch_kt<MAT52>(p, grid, st);
  if (rc || nsplit == 1) return rc;
  const int64_t cnt = p.nrows * p.k;
  f64_reduce_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(p, (int)nsplit);
  KGP_LAUNCH("f64_reduce_kernel");
  return KGP_OK;
}

}  // namespace kgp
