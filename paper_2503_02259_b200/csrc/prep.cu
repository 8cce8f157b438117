#include <cuda_bf16.h>
// Operand preparation for the tcgen05 operator (O(n (d + k)) work per call).
//
// Point data are mean-centred in fp64 and then rounded to fp32 (SURVEY.md §7,
// "Precision": the clamp-at-zero expansion of _panels_numpy.py:19-28 loses
// accuracy on uncentred data). The kernel scale gamma is folded in so the tile
// kernel evaluates t2 = gamma r^2 directly:
//   Gaussian gamma = log2(e) / (2 l^2)   (kappa = 2^-t2)
//   Matern32 gamma = 3 / l^2             (t = sqrt(t2) = sqrt(3) r / l)
//   Matern52 gamma = 5 / l^2
// expansion form (d > 4): t2 = q_i + q_j + sum_k u_ik v_jk, q = gamma |c|^2,
//                         u = -2 gamma c (rows), v = c (columns)
// direct form   (d <= 4): t2 = sum_k (v_jk - u_ik)^2, u = v = sqrt(gamma) c
#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

__host__ __device__ inline double kernel_gamma(int kt, double l) {
  if (kt == GAUSS) return LOG2E / (2.0 * l * l);
  if (kt == MAT32) return 3.0 / (l * l);
  return 5.0 / (l * l);
}

__global__ void col_mean_kernel(int64_t n, int d, const double* __restrict__ x, double* __restrict__ mean) {
  const int k = blockIdx.x;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += x[i * d + k];
  __shared__ double red[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) mean[k] = v / (double)n;
  }
}

__global__ void prep_rows_kernel(int kt, int d, int dpad, bool direct, int64_t nrows, const double* __restrict__ x,
                                 const double* __restrict__ mean, double gamma, float* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  float* o = out + i * (dpad + 1);
  double sg = sqrt(gamma), nrm = 0.0;
  for (int k = 0; k < dpad; ++k) {
    double c = (k < d) ? x[i * d + k] - mean[k] : 0.0;
    nrm += c * c;
    o[1 + k] = direct ? (float)(sg * c) : (float)(-2.0 * gamma * c);
  }
  o[0] = direct ? 0.0f : (float)(gamma * nrm);
}

__global__ void prep_cols_kernel(int kt, int d, int dpad, int mode, int64_t n, int nblk,
                                 const double* __restrict__ x, const double* __restrict__ mean, double gamma,
                                 float* __restrict__ out) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= (int64_t)nblk * 32) return;
  const int64_t t = j >> 5;
  const int jj = (int)(j & 31);
  double c[16], nrm = 0.0;
  for (int k = 0; k < dpad; ++k) {
    c[k] = (j < n && k < d) ? x[j * d + k] - mean[k] : 0.0;
    nrm += c[k] * c[k];
  }
  if (mode != 1) {
    // position inside the block: the tile kernel's thread g reads columns
    // 2g + {0, 1} + 8m (m < 4) as two float4 at 8g
    // mode 0 (direct differences): [0 | sqrt(gamma) c_j]; mode 2 (FP32 expansion): [gamma |c_j|^2 | c_j]
    const int m = jj >> 3, cc = jj & 7;
    const int pos = 8 * (cc >> 1) + 2 * m + (cc & 1);
    float* o = out + t * (int64_t)(dpad + 1) * 32;
    const double sg = mode == 0 ? sqrt(gamma) : 1.0;
    for (int k = 0; k < dpad; ++k) o[(1 + k) * 32 + pos] = (float)(sg * c[k]);
    o[pos] = mode == 0 ? 0.0f : (float)(gamma * nrm);
    return;
  }
  // tensor-core distance (kgp_common.cuh tc_dist_kd): V'_j = [c_j (dpad), 1, 1, q_j hi, q_j lo, 0 ...]
  // (KGP_TC_DIST4; else [c_j, 1, q_j, 0 ...]) as tf32 hi / lo tiles (K-major, no swizzle, 32 rows),
  // block t at byte t * 2 * 32 * kd * 4
  const int kd = tc_dist_kd(dpad);
  uint8_t* base = reinterpret_cast<uint8_t*>(out) + t * (int64_t)(2 * 32 * kd * 4);
  const double q = gamma * nrm;
  const float qf = (float)q;
  const float qh = __uint_as_float(__float_as_uint(qf) & 0xFFFFE000u);
  const float ql = (float)(q - (double)qh);
  for (int k = 0; k < kd; ++k) {
    float v = 0.0f;
    if (KGP_TC_DIST4) {
      if (j < n) v = (k < dpad) ? (float)c[k] : (k == dpad || k == dpad + 1) ? 1.0f : k == dpad + 2 ? qh : k == dpad + 3 ? ql : 0.0f;
    } else {
      if (j < n) v = (k < dpad) ? (float)c[k] : (k == dpad ? 1.0f : (k == dpad + 1 ? qf : 0.0f));
    }
    const bool split = !KGP_TC_DIST4 || k < dpad;
    const float hi = split ? __uint_as_float(__float_as_uint(v) & 0xFFFFE000u) : v;
    const uint32_t off = interleave_offset((uint32_t)jj, (uint32_t)k, 32);
    *reinterpret_cast<float*>(base + off) = hi;
    *reinterpret_cast<float*>(base + 32 * kd * 4 + off) = split ? v - hi : 0.0f;
  }
}

__device__ inline uint32_t tf32_rna_bits(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}

__global__ void prep_rhs_kernel(int split, int lb, int64_t n, int64_t k, int64_t c0, int kp, int blk0, int nblk,
                                const double* __restrict__ b, int64_t b_rs, int64_t b_cs, uint8_t* __restrict__ out) {
  // one thread per (block t, rhs column c, in-block row jj); jj fastest for coalesced column-major reads;
  // blocks [blk0, blk0 + nblk)
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)nblk * kp * 32;
  if (g >= total) return;
  const int jj = (int)(g & 31);
  const int c = (int)((g >> 5) % kp);
  const int64_t t = blk0 + (g >> 5) / kp;
  const int64_t j = t * 32 + jj;
  const int64_t cc = c0 + c;
  double v = (j < n && cc < k) ? b[j * b_rs + cc * b_cs] : 0.0;
  const int tpo = (split == 3) ? 2 : 1;
  uint8_t* tile = out + t * (int64_t)(tpo * 128 + (lb ? 64 : 0)) * kp;
  const uint32_t off = sw128_offset((uint32_t)c, (uint32_t)jj);
  float vf = (float)v;
  if (split == 2) {
    // bf16x3: B = B0 + B1 (two round-to-nearest bf16 terms), each in the interleaved K-major
    // layout of the kind::f16 B operand: B0 at +0, B1 at +64 kp
    const __nv_bfloat16 b0 = __float2bfloat16_rn(vf);
    const __nv_bfloat16 b1 = __float2bfloat16_rn(vf - __bfloat162float(b0));
    const uint32_t o16 = interleave16_offset((uint32_t)c, (uint32_t)jj, (uint32_t)kp);
    *reinterpret_cast<__nv_bfloat16*>(tile + o16) = b0;
    *reinterpret_cast<__nv_bfloat16*>(tile + 64 * kp + o16) = b1;
  } else if (split == 3) {
    uint32_t hi = __float_as_uint(vf) & 0xFFFFE000u;
    float lo = vf - __uint_as_float(hi);
    *reinterpret_cast<uint32_t*>(tile + off) = hi;
    *reinterpret_cast<float*>(tile + kp * 128 + off) = lo;
    // lb: + bf16(B) in the interleaved K-major layout (B operand of the bf16 lo*hi correction)
    if (lb) *reinterpret_cast<__nv_bfloat16*>(tile + 2 * kp * 128 + interleave16_offset((uint32_t)c, (uint32_t)jj, (uint32_t)kp)) = __float2bfloat16_rn(vf);
  } else {
    *reinterpret_cast<uint32_t*>(tile + off) = tf32_rna_bits(vf);
  }
}

}  // namespace

int col_mean(int64_t n, int d, const double* x, double* mean, cudaStream_t st) {
  col_mean_kernel<<<d, 256, 0, st>>>(n, d, x, mean);
  KGP_LAUNCH("col_mean_kernel");
  return KGP_OK;
}

int prep_rows(int kt, int /*split*/, int d, int dpad, int64_t nrows, const double* x, const double* mean, double l,
              float* out, cudaStream_t st) {
  if (nrows <= 0) return KGP_OK;
  prep_rows_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(kt, d, dpad, tc_direct(dpad), nrows, x, mean,
                                                                     kernel_gamma(kt, l), out);
  KGP_LAUNCH("prep_rows_kernel");
  return KGP_OK;
}

int prep_cols(int kt, int d, int dpad, int64_t n, const double* x, const double* mean, double l, float* out,
              cudaStream_t st) {
  int nblk = (int)((n + 31) / 32);
  int64_t tot = (int64_t)nblk * 32;
  prep_cols_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(kt, d, dpad, tc_dist_mode(dpad), n, nblk, x, mean,
                                                                    kernel_gamma(kt, l), out);
  KGP_LAUNCH("prep_cols_kernel");
  return KGP_OK;
}

int prep_rhs(int split, int lb, int64_t n, int64_t k, int64_t c0, int kp, const double* b, int64_t b_rs, int64_t b_cs,
             uint8_t* out, cudaStream_t st, int blk0, int blk1) {
  const int nall = (int)((n + 31) / 32);
  if (blk1 < 0 || blk1 > nall) blk1 = nall;
  const int nblk = blk1 - blk0;
  if (nblk <= 0) return KGP_OK;
  int64_t total = (int64_t)nblk * kp * 32;
  prep_rhs_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(split, lb, n, k, c0, kp, blk0, nblk, b, b_rs, b_cs,
                                                                    out);
  KGP_LAUNCH("prep_rhs_kernel");
  return KGP_OK;
}

double tc_kernel_gamma(int kt, double l) { return kernel_gamma(kt, l); }

}  // namespace kgp
