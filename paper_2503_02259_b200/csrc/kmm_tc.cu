// Fused kernel-matrix MatMul on the 5th-generation tensor cores (sm_100a).
//
// Replaces KernelEngine._streamed_matmul (kmat.py:165-189) and the numba panels
// (_panels_numba.py:37-131) for precision KGP_FAST / KGP_TF32:
//
//   acc_K  = kappa(X_rows, X) . B        acc_G = (scaled dkappa/dl)(X_rows, X) . B
//
// The kernel matrix is never stored. Per CTA: 128 rows (TMEM lanes). The column
// dimension j streams in blocks of 32:
//   * a producer warp bulk-copies (cp.async.bulk) the block's RHS tiles (pre-split
//     into tf32 hi/lo, already in the UMMA 128B-swizzled K-major layout) and the
//     block's column-point data into a 4-stage shared-memory ring;
//   * 8 compute warps evaluate the 128x32 tile in registers (fp32, centred
//     coordinates, packed FFMA2 for the distance, MUFU ex2/sqrt for the
//     transform) and store it, split into tf32 hi/lo, straight into TMEM
//     (tcgen05.st) -- the A operand of the MMA;
//   * one thread issues tcgen05.mma kind::tf32 (A from TMEM, B from shared
//     memory, D in TMEM): 3 MMAs per output per K=8 chunk for 3xTF32.
// The accumulators stay in TMEM for the whole row sweep; the epilogue applies
// f^2, 2f, s*B and the derivative scale in fp64 and writes the outputs.
#include <cuda.h>

#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

constexpr int NCW = 8;        // compute warps
constexpr int NTHREADS = (NCW + 2) * 32;
constexpr int NSB = 4;        // shared-memory ring depth (RHS + column data)
constexpr int BJ = 32;        // columns per block (one 128-byte swizzle atom of tf32)

KGP_DEV float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
KGP_DEV float sqrtf_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
KGP_DEV uint32_t tf32_hi_bits(float v) { return __float_as_uint(v) & 0xFFFFE000u; }

// kernel transform of the scaled squared distance t2 (see prep kernels for the
// per-kernel scale gamma):   Gaussian t2 = r^2 log2(e)/(2 l^2),  kappa = 2^-t2
//                            Matern32 t2 = 3 r^2 / l^2,           kappa = (1+t) e^-t
//                            Matern52 t2 = 5 r^2 / l^2,           kappa = (1+t+t2/3) e^-t
// and g = t2 * (d kappa / d t2-ish factor) so that dkappa/dl = scale_dl * g.
template <int KT, bool NEED_G>
KGP_DEV void transform(float t2, float& kv, float& gv) {
  t2 = fmaxf(t2, 0.0f);  // the expansion can cancel below zero (_panels_numpy.py:26-27)
  if (KT == GAUSS) {
    float e = ex2f(-t2);
    kv = e;
    if (NEED_G) gv = t2 * e;
  } else {
    float t = sqrtf_approx(t2);
    float e = ex2f(-1.4426950408889634f * t);
    float u = fmaf(t, e, e);  // (1+t) e^-t
    if (KT == MAT32) {
      kv = u;
      if (NEED_G) gv = t2 * e;
    } else {
      kv = fmaf(t2 * (1.0f / 3.0f), e, u);
      if (NEED_G) gv = t2 * u;
    }
  }
}

template <int KT, int D, bool DIRECT, int NOUT, int SPLIT>
__global__ void __launch_bounds__(NTHREADS, 1) kmm_tc_kernel(const TcParams p) {
  constexpr int TPO = (SPLIT == 3) ? 2 : 1;  // TMEM tiles per output (hi, lo)
  constexpr int ATILES = NOUT * TPO;
  constexpr int XFL = (D + 1) * BJ;          // floats of column data per block
  constexpr uint32_t XBYTES = XFL * 4;
  constexpr bool NEED_G = (NOUT == 2);

  extern __shared__ __align__(1024) uint8_t smem[];
  const int KP = p.kp;
  const uint32_t BBYTES = (uint32_t)(TPO * KP * 128);
  uint8_t* sB = smem;                                   // NSB x BBYTES, 1024-aligned
  float* sX = reinterpret_cast<float*>(smem + NSB * BBYTES);  // NSB x XFL
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSB * BBYTES + NSB * XBYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSB;
  uint64_t* afull = bars + 2 * NSB;
  uint64_t* aempty = bars + 2 * NSB + 4;
  uint64_t* accfull = bars + 2 * NSB + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NSB + 9);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int NSA = p.nsa;
  const int abase = 512 - NSA * ATILES * 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + NCW);
    }
    for (int a = 0; a < NSA; ++a) {
      mbar_init(&afull[a], NCW);
      mbar_init(&aempty[a], 1);
    }
    mbar_init(accfull, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int nblk = p.nblk;

  if (warp == NCW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint8_t* gB = p.bsplit;
      const float* gX = p.xcol;
      for (int t = 0; t < nblk; ++t) {
        const int s = t % NSB;
        mbar_wait(&empty[s], ((t / NSB) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], BBYTES + XBYTES);
        bulk_g2s(sB + s * BBYTES, gB + (size_t)t * BBYTES, BBYTES, &full[s]);
        bulk_g2s(sX + s * XFL, gX + (size_t)t * XFL, XBYTES, &full[s]);
      }
    }
  } else if (warp == NCW + 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32_m128(KP);
      for (int t = 0; t < nblk; ++t) {
        const int s = t % NSB;
        const int a = t % NSA;
        mbar_wait(&full[s], (t / NSB) & 1);
        mbar_wait(&afull[a], (t / NSA) & 1);
        tc_fence_after();
        const uint32_t bhi = smem_u32(sB + s * BBYTES);
        const uint64_t dhi = sw128_kmajor_desc(bhi);
        const uint64_t dlo = sw128_kmajor_desc(bhi + KP * 128);
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
          const uint32_t dt = tbase + o * KP;
          const uint32_t ahi = tbase + abase + (a * ATILES + o * TPO) * 32;
#pragma unroll
          for (int kk = 0; kk < BJ / 8; ++kk) {
            const uint32_t acc = (t > 0 || kk > 0) ? 1u : 0u;
            mma_tf32_ts(dt, ahi + 8 * kk, dhi + 2 * kk, idesc, acc);
            if (SPLIT == 3) {
              mma_tf32_ts(dt, ahi + 8 * kk, dlo + 2 * kk, idesc, 1u);
              mma_tf32_ts(dt, ahi + 32 + 8 * kk, dhi + 2 * kk, idesc, 1u);
            }
          }
        }
        tc_commit(&empty[s]);
        tc_commit(&aempty[a]);
      }
      tc_commit(accfull);
    }
  } else {
    // ------------------------------------------------------------ compute warps
    const int qd = warp & 3;   // TMEM lane quadrant
    const int h = warp >> 2;   // which 16 of the 32 block columns
    const int64_t r = (int64_t)blockIdx.x * 128 + qd * 32 + lane;
    float qi = 0.f, u[D];
    if (r < p.nrows) {
      const float* xr = p.xrow + r * (D + 1);
      qi = xr[0];
#pragma unroll
      for (int k = 0; k < D; ++k) u[k] = xr[1 + k];
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) u[k] = 0.f;
    }
    const uint32_t lane_base = tbase + ((uint32_t)(qd * 32) << 16);
    for (int t = 0; t < nblk; ++t) {
      const int s = t % NSB;
      const int a = t % NSA;
      mbar_wait(&full[s], (t / NSB) & 1);
      const float* xs = sX + s * XFL + 16 * h;
      float2 acc[8];
      if (DIRECT) {
#pragma unroll
        for (int pq = 0; pq < 8; ++pq) acc[pq] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float4* v4 = reinterpret_cast<const float4*>(xs + (k + 1) * BJ);
          const float2 uk = make_float2(-u[k], -u[k]);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            float4 v = v4[q4];
            float2 d0 = __fadd2_rn(make_float2(v.x, v.y), uk);
            float2 d1 = __fadd2_rn(make_float2(v.z, v.w), uk);
            acc[2 * q4] = __ffma2_rn(d0, d0, acc[2 * q4]);
            acc[2 * q4 + 1] = __ffma2_rn(d1, d1, acc[2 * q4 + 1]);
          }
        }
      } else {
        const float4* q4p = reinterpret_cast<const float4*>(xs);
        const float2 qq = make_float2(qi, qi);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float4 v = q4p[q4];
          acc[2 * q4] = __fadd2_rn(make_float2(v.x, v.y), qq);
          acc[2 * q4 + 1] = __fadd2_rn(make_float2(v.z, v.w), qq);
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float4* v4 = reinterpret_cast<const float4*>(xs + (k + 1) * BJ);
          const float2 uk = make_float2(u[k], u[k]);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            float4 v = v4[q4];
            acc[2 * q4] = __ffma2_rn(uk, make_float2(v.x, v.y), acc[2 * q4]);
            acc[2 * q4 + 1] = __ffma2_rn(uk, make_float2(v.z, v.w), acc[2 * q4 + 1]);
          }
        }
      }
      // column data consumed: release this ring slot for the producer
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);

      uint32_t kh[16], kl[16], gh[16], gl[16];
#pragma unroll
      for (int pq = 0; pq < 8; ++pq) {
        float k0, k1, g0 = 0.f, g1 = 0.f;
        transform<KT, NEED_G>(acc[pq].x, k0, g0);
        transform<KT, NEED_G>(acc[pq].y, k1, g1);
        if (SPLIT == 3) {
          kh[2 * pq] = tf32_hi_bits(k0);
          kh[2 * pq + 1] = tf32_hi_bits(k1);
          kl[2 * pq] = __float_as_uint(k0 - __uint_as_float(kh[2 * pq]));
          kl[2 * pq + 1] = __float_as_uint(k1 - __uint_as_float(kh[2 * pq + 1]));
          if (NEED_G) {
            gh[2 * pq] = tf32_hi_bits(g0);
            gh[2 * pq + 1] = tf32_hi_bits(g1);
            gl[2 * pq] = __float_as_uint(g0 - __uint_as_float(gh[2 * pq]));
            gl[2 * pq + 1] = __float_as_uint(g1 - __uint_as_float(gh[2 * pq + 1]));
          }
        } else {
          kh[2 * pq] = __float_as_uint(k0);
          kh[2 * pq + 1] = __float_as_uint(k1);
          if (NEED_G) {
            gh[2 * pq] = __float_as_uint(g0);
            gh[2 * pq + 1] = __float_as_uint(g1);
          }
        }
      }
      // wait until the MMAs that read this A stage NSA blocks ago have finished
      mbar_wait(&aempty[a], ((t / NSA) & 1) ^ 1);
      tc_fence_after();
      const uint32_t ta = lane_base + abase + a * ATILES * 32 + 16 * h;
      tmem_st16(ta, kh);
      if (SPLIT == 3) tmem_st16(ta + 32, kl);
      if (NEED_G) {
        tmem_st16(ta + TPO * 32, gh);
        if (SPLIT == 3) tmem_st16(ta + TPO * 32 + 32, gl);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[a]);
    }

    // ------------------------------------------------------------ epilogue
    mbar_wait(accfull, 0);
    tc_fence_after();
    // columns of the accumulator region handled by this warp: NOUT*KP split in two halves
    // 16-column chunks of the NOUT*KP accumulator columns alternate between the
    // two warps of a lane quadrant (KP is a multiple of 16: no chunk straddles outputs)
    const int total = NOUT * KP;
    for (int cb = 16 * h; cb < total; cb += 32) {
      uint32_t v[16];
      tmem_ld16(lane_base + cb, v);
      tc_wait_ld();
      if (r >= p.nrows) continue;
      const int o = cb / KP;
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int c = cb - o * KP + jj;
        if (c >= p.k) continue;
        const double a = (double)__uint_as_float(v[jj]);
        if (o == 0) {
          if (p.out_k) {
            double val = p.f2 * a;
            if (p.diag_row0 >= 0) val += p.s * p.b[(p.diag_row0 + r) * p.b_rs + c * p.b_cs];
            p.out_k[r * p.o_rs + c * p.o_cs] = val;
          }
          if (p.out_df) p.out_df[r * p.o_rs + c * p.o_cs] = p.two_f * a;
        } else if (p.out_dl) {
          p.out_dl[r * p.o_rs + c * p.o_cs] = p.scale_dl * a;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int KT, int D, bool DIRECT, int NOUT, int SPLIT>
int launch_one(const TcParams& p, cudaStream_t st) {
  auto kern = kmm_tc_kernel<KT, D, DIRECT, NOUT, SPLIT>;
  const int TPO = (SPLIT == 3) ? 2 : 1;
  size_t smem = NSB * (size_t)(TPO * p.kp * 128) + NSB * (size_t)((D + 1) * BJ * 4) + 256;
  static bool configured = false;  // one attribute call per instantiation
  if (!configured) {
    KGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  dim3 grid((unsigned)((p.nrows + 127) / 128));
  kern<<<grid, NTHREADS, smem, st>>>(p);
  KGP_LAUNCH("kmm_tc_kernel");
  return KGP_OK;
}

template <int KT, int D, bool DIRECT>
int launch_kt_d(const TcParams& p, int nout, int split, cudaStream_t st) {
  if (nout == 1) return split == 3 ? launch_one<KT, D, DIRECT, 1, 3>(p, st) : launch_one<KT, D, DIRECT, 1, 1>(p, st);
  return split == 3 ? launch_one<KT, D, DIRECT, 2, 3>(p, st) : launch_one<KT, D, DIRECT, 2, 1>(p, st);
}

template <int KT>
int launch_kt(const TcParams& p, int dpad, int nout, int split, cudaStream_t st) {
  switch (dpad) {
    case 2: return launch_kt_d<KT, 2, true>(p, nout, split, st);
    case 4: return launch_kt_d<KT, 4, true>(p, nout, split, st);
    case 8: return launch_kt_d<KT, 8, false>(p, nout, split, st);
    case 16: return launch_kt_d<KT, 16, false>(p, nout, split, st);
  }
  set_error(KGP_ERR_INVALID, "fast path supports d <= 16");
  return KGP_ERR_INVALID;
}

}  // namespace

int tc_pad_dim(int d) { return d <= 2 ? 2 : d <= 4 ? 4 : d <= 8 ? 8 : 16; }
bool tc_direct(int dpad) { return dpad <= 4; }

int launch_kmm_tc(int kt, int dpad, int nout, int split, const TcParams& p, cudaStream_t st) {
  switch (kt) {
    case GAUSS: return launch_kt<GAUSS>(p, dpad, nout, split, st);
    case MAT32: return launch_kt<MAT32>(p, dpad, nout, split, st);
    case MAT52: return launch_kt<MAT52>(p, dpad, nout, split, st);
  }
  set_error(KGP_ERR_INVALID, "unknown kernel id %d", kt);
  return KGP_ERR_INVALID;
}

}  // namespace kgp
