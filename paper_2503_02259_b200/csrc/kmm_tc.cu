// Fused kernel-matrix MatMul on the 5th-generation tensor cores (sm_100a).
//
// Replaces KernelEngine._streamed_matmul (kmat.py:165-189) and the numba panels
// (_panels_numba.py:37-131) for precision KGP_FAST / KGP_TF32:
//
//   acc_K = kappa(X_rows, X) . B        acc_G = (scaled dkappa/dl)(X_rows, X) . B
//
// The kernel matrix is never stored. One CTA owns 128 rows (the TMEM lanes) and
// streams the columns in blocks of 32 (one 128-byte swizzle atom of tf32):
//   * warp 8 (producer) bulk-copies each block's RHS tiles -- pre-split into tf32
//     hi/lo and already in the UMMA K-major 128B-swizzled layout -- and the
//     block's column-point data into a 4-stage shared-memory ring;
//   * warps 0-7 (compute) evaluate the 128x32 tile in registers: fp32 centred
//     coordinates, packed FFMA2 distances, MUFU ex2/sqrt transforms; each thread
//     owns a 4-row x 4-column patch so one broadcast LDS.128 of column data feeds
//     16 FMAs. The tile, split into tf32 hi/lo, goes straight to TMEM
//     (tcgen05.st 16x256b): the A operand of the MMA;
//   * warp 9 issues tcgen05.mma kind::tf32 (A in TMEM, B in shared memory,
//     D in TMEM): hi*hi + hi*lo + lo*hi per output and K=8 chunk for 3xTF32;
//   * warps 10-13 (drain) promote the TMEM accumulators every `flush` blocks into
//     fp32 shared-memory sums (two accumulator buffers ping-pong, so the MMA never
//     waits). The tensor core's fp32 accumulation truncates; unpromoted it drifts
//     linearly in n (measured 4.6e-4 at n=65536), promoted it stays near 1e-6.
// The drain warps then apply f^2, 2f, s*B and the derivative scale in fp64 and
// write the outputs.
#include <cuda.h>

#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

constexpr int NCW = 8;                    // compute warps (2 per TMEM lane quadrant)
constexpr int WPROD = NCW, WMMA = NCW + 1;
constexpr int NTHREADS = (NCW + 6) * 32;  // + producer, MMA, 4 drain warps = 448
constexpr int NSB = 4;                    // shared-memory ring depth (RHS + column data)
constexpr int BJ = 32;                    // columns per block

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
KGP_DEV float2 hi2(float2 v) {
  return make_float2(__uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
}
KGP_DEV float2 fsub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
KGP_DEV float2 lo2(float2 v) { return fsub2(v, hi2(v)); }

// Kernel transform of the scaled squared distance t2 = gamma r^2 (see prep.cu):
//   Gaussian  t2 = r^2 log2(e) / (2 l^2)   kappa = 2^-t2              g = t2 kappa
//   Matern32  t2 = 3 r^2 / l^2             kappa = (1+t) e^-t         g = t2 e^-t
//   Matern52  t2 = 5 r^2 / l^2             kappa = (1+t+t2/3) e^-t    g = t2 (1+t) e^-t
// with t = sqrt(t2); dkappa/dl = scale_dl * g (scale folded into the epilogue).
template <int KT, bool NEED_G>
KGP_DEV void transform2(float2 t2, float2& kv, float2& gv) {
  t2.x = fmaxf(t2.x, 0.0f);  // the expansion can cancel below zero (_panels_numpy.py:26-27)
  t2.y = fmaxf(t2.y, 0.0f);
  if (KT == GAUSS) {
    kv = make_float2(ex2f(-t2.x), ex2f(-t2.y));
    if (NEED_G) gv = __fmul2_rn(t2, kv);
  } else {
    float2 t = make_float2(sqrtf_approx(t2.x), sqrtf_approx(t2.y));
    float2 a = __fmul2_rn(t, make_float2(-1.4426950408889634f, -1.4426950408889634f));
    float2 e = make_float2(ex2f(a.x), ex2f(a.y));
    float2 u = __ffma2_rn(t, e, e);  // (1+t) e^-t
    if (KT == MAT32) {
      kv = u;
      if (NEED_G) gv = __fmul2_rn(t2, e);
    } else {
      kv = __ffma2_rn(__fmul2_rn(t2, make_float2(1.0f / 3.0f, 1.0f / 3.0f)), e, u);
      if (NEED_G) gv = __fmul2_rn(t2, u);
    }
  }
}

// register order of tcgen05.st 16x256b.x2 for one thread: rows (r, r+8) x column pairs (c, c+8)
KGP_DEV void pack8(uint32_t (&w)[8], float2 r0c0, float2 r1c0, float2 r0c1, float2 r1c1) {
  w[0] = __float_as_uint(r0c0.x); w[1] = __float_as_uint(r0c0.y);
  w[2] = __float_as_uint(r1c0.x); w[3] = __float_as_uint(r1c0.y);
  w[4] = __float_as_uint(r0c1.x); w[5] = __float_as_uint(r0c1.y);
  w[6] = __float_as_uint(r1c1.x); w[7] = __float_as_uint(r1c1.y);
}

template <int SPLIT>
KGP_DEV void store_tile(uint32_t taddr, const float2 (&v)[2][2]) {
  uint32_t w[8];
  if (SPLIT == 3) {
    pack8(w, hi2(v[0][0]), hi2(v[1][0]), hi2(v[0][1]), hi2(v[1][1]));
    tmem_st_16x256b_x2(taddr, w);
    pack8(w, lo2(v[0][0]), lo2(v[1][0]), lo2(v[0][1]), lo2(v[1][1]));
    tmem_st_16x256b_x2(taddr + 32, w);
  } else {
    pack8(w, v[0][0], v[1][0], v[0][1], v[1][1]);
    tmem_st_16x256b_x2(taddr, w);
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
  const int NACC = NOUT * KP;                      // accumulator columns per buffer
  const uint32_t BBYTES = (uint32_t)(TPO * KP * 128);
  uint8_t* sB = smem;                              // NSB x BBYTES, 1024-aligned
  float* sX = reinterpret_cast<float*>(smem + NSB * BBYTES);  // NSB x XFL
  float* sAcc = sX + NSB * XFL;                    // NACC x 128 fp32, column-major
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAcc + NACC * 128);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSB;
  uint64_t* afull = bars + 2 * NSB;
  uint64_t* aempty = bars + 2 * NSB + 4;
  uint64_t* accfull = bars + 2 * NSB + 8;
  uint64_t* accempty = bars + 2 * NSB + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NSB + 12);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int NSA = p.nsa;
  const int abase = 2 * NACC;  // A stages follow the two accumulator buffers
  const int nblk = p.nblk;
  const int flush = p.flush;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + NCW);
    }
    for (int a = 0; a < NSA; ++a) {
      mbar_init(&afull[a], NCW);
      mbar_init(&aempty[a], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == WPROD) {
    // ------------------------------------------------------------ producer (converged warp, one elected issuer)
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0; t < nblk; ++t) {
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(&full[s], BBYTES + XBYTES);
        bulk_g2s(sB + s * BBYTES, p.bsplit + (size_t)t * BBYTES, BBYTES, &full[s]);
        bulk_g2s(sX + s * XFL, p.xcol + (size_t)t * XFL, XBYTES, &full[s]);
      }
      __syncwarp();
      if (++s == NSB) { s = 0; ph ^= 1; }
    }
  } else if (warp == WMMA) {
    // ------------------------------------------------------------ MMA issuer (converged warp, one elected issuer)
    const uint32_t idesc = idesc_tf32_m128(KP);
    int s = 0, a = 0, pos = 0, ab = 0;
    uint32_t ph_s = 0, ph_a = 0, ph_acc = 0;
    for (int t = 0; t < nblk; ++t) {
      if (pos == 0) mbar_wait(&accempty[ab], ph_acc ^ 1);  // buffer drained (segment start)
      mbar_wait(&full[s], ph_s);
      mbar_wait(&afull[a], ph_a);
      tc_fence_after();
      const uint32_t bhi = smem_u32(sB + s * BBYTES);
      const uint64_t dhi = sw128_kmajor_desc(bhi);
      const uint64_t dlo = sw128_kmajor_desc(bhi + KP * 128);
      const bool last = (pos + 1 == flush) || (t == nblk - 1);
      if (elect_one()) {
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
          const uint32_t dt = tbase + ab * NACC + o * KP;
          const uint32_t ahi = tbase + abase + (a * ATILES + o * TPO) * 32;
#pragma unroll
          for (int kk = 0; kk < BJ / 8; ++kk) {
            const uint32_t acc = (pos > 0 || kk > 0) ? 1u : 0u;
            mma_tf32_ts(dt, ahi + 8 * kk, dhi + 2 * kk, idesc, acc);
            if (SPLIT == 3) {
              mma_tf32_ts(dt, ahi + 8 * kk, dlo + 2 * kk, idesc, 1u);
              mma_tf32_ts(dt, ahi + 32 + 8 * kk, dhi + 2 * kk, idesc, 1u);
            }
          }
        }
        tc_commit(&empty[s]);
        tc_commit(&aempty[a]);
        if (last) tc_commit(&accfull[ab]);
      }
      __syncwarp();
      if (last) {
        pos = 0;
        if (ab == 1) ph_acc ^= 1;
        ab ^= 1;
      } else {
        ++pos;
      }
      if (++s == NSB) { s = 0; ph_s ^= 1; }
      if (++a == NSA) { a = 0; ph_a ^= 1; }
    }
  } else if (warp < NCW) {
    // ------------------------------------------------------------ compute warps
    const int qd = warp & 3;  // TMEM lane quadrant
    const int h = warp >> 2;  // columns [16h, 16h+16) of each block
    const int g = lane & 3;
    // rows owned by this thread: 32 qd + lane/4 + {0, 8, 16, 24}
    float qi[4], u[4][D];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int64_t r = (int64_t)blockIdx.x * 128 + qd * 32 + (lane >> 2) + 8 * rr;
      const bool ok = r < p.nrows;
      const float* xr = p.xrow + (ok ? r : 0) * (D + 1);
      qi[rr] = ok ? xr[0] : 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) u[rr][k] = ok ? xr[1 + k] : 0.f;
    }
    const uint32_t lane_base = tbase + ((uint32_t)(qd * 32) << 16);
    int s = 0, a = 0, prev_a = -1;
    uint32_t ph_s = 0, ph_a = 0;
    for (int t = 0; t < nblk; ++t) {
      mbar_wait(&full[s], ph_s);
      // this thread's columns, permuted by prep_cols: (c, c+1, c+8, c+9), c = 16h + 2g
      const float* xs = sX + s * XFL + 16 * h + 4 * g;
      float2 acc[4][2];  // [row][column pair]
      if (DIRECT) {
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) acc[rr][0] = acc[rr][1] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float4 v = *reinterpret_cast<const float4*>(xs + (k + 1) * BJ);
          const float2 v0 = make_float2(v.x, v.y), v1 = make_float2(v.z, v.w);
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const float2 uk = make_float2(u[rr][k], u[rr][k]);
            const float2 d0 = fsub2(v0, uk);
            const float2 d1 = fsub2(v1, uk);
            acc[rr][0] = __ffma2_rn(d0, d0, acc[rr][0]);
            acc[rr][1] = __ffma2_rn(d1, d1, acc[rr][1]);
          }
        }
      } else {
        const float4 qv = *reinterpret_cast<const float4*>(xs);
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const float2 qq = make_float2(qi[rr], qi[rr]);
          acc[rr][0] = __fadd2_rn(make_float2(qv.x, qv.y), qq);
          acc[rr][1] = __fadd2_rn(make_float2(qv.z, qv.w), qq);
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float4 v = *reinterpret_cast<const float4*>(xs + (k + 1) * BJ);
          const float2 v0 = make_float2(v.x, v.y), v1 = make_float2(v.z, v.w);
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const float2 uk = make_float2(u[rr][k], u[rr][k]);
            acc[rr][0] = __ffma2_rn(uk, v0, acc[rr][0]);
            acc[rr][1] = __ffma2_rn(uk, v1, acc[rr][1]);
          }
        }
      }
      // column data consumed: release the ring slot
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      // hand the previous block's A stage to the MMA (its stores were issued one block ago)
      if (prev_a >= 0) {
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[prev_a]);
      }
      mbar_wait(&aempty[a], ph_a ^ 1);
      tc_fence_after();
      const uint32_t tcol = lane_base + abase + a * ATILES * 32 + 16 * h;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        // 16-lane group `half`: this thread's rows lane/4 (+16 half) and lane/4 + 8
        float2 kv[2][2], gv[2][2];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int cp = 0; cp < 2; ++cp) transform2<KT, NEED_G>(acc[2 * half + q][cp], kv[q][cp], gv[q][cp]);
        const uint32_t taddr = tcol + ((uint32_t)(16 * half) << 16);
        store_tile<SPLIT>(taddr, kv);
        if (NEED_G) store_tile<SPLIT>(taddr + TPO * 32, gv);
      }
      prev_a = a;
      if (++s == NSB) { s = 0; ph_s ^= 1; }
      if (++a == NSA) { a = 0; ph_a ^= 1; }
    }
    if (prev_a >= 0) {
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[prev_a]);
    }
  } else {
    // ------------------------------------------------------------ drain + epilogue warps
    const int qd = warp & 3;
    const int row = qd * 32 + lane;
    const uint32_t lane_base = tbase + ((uint32_t)(qd * 32) << 16);
    const int nseg = (nblk + flush - 1) / flush;
    int ab = 0;
    uint32_t ph = 0;
    for (int seg = 0; seg < nseg; ++seg) {
      mbar_wait(&accfull[ab], ph);
      tc_fence_after();
      for (int cb = 0; cb < NACC; cb += 16) {
        uint32_t v[16];
        tmem_ld16(lane_base + ab * NACC + cb, v);
        tc_wait_ld();
        float* dst = sAcc + cb * 128 + row;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const float x = __uint_as_float(v[jj]);
          dst[jj * 128] = (seg == 0) ? x : dst[jj * 128] + x;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[ab]);
      if (ab == 1) ph ^= 1;
      ab ^= 1;
    }
    // epilogue: fp64 scaling, + s B on the diagonal rows, strided writes
    const int64_t r = (int64_t)blockIdx.x * 128 + row;
    if (r < p.nrows) {
      for (int c = 0; c < p.k; ++c) {
        const double ak = (double)sAcc[c * 128 + row];
        const int64_t o = r * p.o_rs + c * p.o_cs;
        if (p.out_k) {
          double val = p.f2 * ak;
          if (p.diag_row0 >= 0) val += p.s * p.b[(p.diag_row0 + r) * p.b_rs + c * p.b_cs];
          p.out_k[o] = val;
        }
        if (p.out_df) p.out_df[o] = p.two_f * ak;
        if (NEED_G && p.out_dl) p.out_dl[o] = p.scale_dl * (double)sAcc[(KP + c) * 128 + row];
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
  size_t smem = NSB * (size_t)(TPO * p.kp * 128) + NSB * (size_t)((D + 1) * BJ * 4) +
                (size_t)NOUT * p.kp * 128 * 4 + 256;
  KGP_REQUIRE(smem <= 225 * 1024, KGP_ERR_INVALID, "fast operator tile config needs %zu B of shared memory", smem);
  static bool configured = false;  // one attribute call per instantiation
  if (!configured) {
    KGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
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

int tc_max_kp(int nout, int split) {
  // TMEM: two accumulator buffers (2 * nout * kp columns) + at least two A stages
  const int stage = nout * (split == 3 ? 2 : 1) * 32;
  int kp = (512 - 2 * stage) / (2 * nout);
  kp = kp / 16 * 16;
  return kp > 128 ? 128 : kp;
}

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
