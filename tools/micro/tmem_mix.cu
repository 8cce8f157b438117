// Does TMEM store traffic slow the tensor pipe? One CTA per SM; an MMA warp issues the fused
// operator's per-block contraction pattern (2 outputs x 4 K-steps x {hi.hi, hi.lo, lo.hi},
// tf32 M=128 N=32 K=8, A in TMEM, B 128B-swizzled in SMEM) `reps` times, fully unrolled,
// while 0/4/8 warps store (tcgen05.st 32x32b.x16) or load TMEM columns disjoint from the MMA's.
// Variant BF: the bf16 split pattern (2 outputs x 2 K-steps x {A0.B0, A0.B1, A1.B0},
// kind::f16 M=128 N=32 K=16). Prints cycles per rep (= per 32-column block) seen by the MMA warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2503_02259_b200/csrc -o tmem_mix tmem_mix.cu
#include <cstdio>

#include "kgp_common.cuh"

using namespace kgp;

// side: 0 none, 1 stores (64 KB per rep over nside warps), 2 loads (64 KB per rep)
template <bool BF>
__global__ void mix(int reps, int side, int nside, unsigned long long* out, int ncommit) {
  __shared__ __align__(1024) uint8_t sb[2 * 32 * 128];
  __shared__ uint64_t bar;
  __shared__ uint64_t cb[4];
  __shared__ uint32_t slot;
  __shared__ volatile int go;
  for (int i = threadIdx.x; i < 2 * 32 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3f803f80u;
  fence_proxy_async_smem();
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1);
    fence_barrier_init();
    go = 0;
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  const int mma_warp = 8;
  if (warp == mma_warp) {
    const uint32_t idt = idesc_tf32_m128(32), idb = idesc_bf16_m128(32);
    const uint32_t bhi = smem_u32(sb);
    const uint64_t dhi = sw128_kmajor_desc(bhi), dlo = sw128_kmajor_desc(bhi + 32 * 128);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (elect_one()) {
        const uint32_t dt = tbase + 64 * (r & 1);  // two accumulator buffers, 2 outputs x 32 columns
        const uint32_t a = tbase + 128 + 128 * (r & 1);
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          if (!BF) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              mma_tf32_ts(dt + 32 * o, a + 64 * o + 8 * kk, dhi + 2 * kk, idt, kk > 0 ? 1u : 0u);
              mma_tf32_ts(dt + 32 * o, a + 64 * o + 8 * kk, dlo + 2 * kk, idt, 1u);
              mma_tf32_ts(dt + 32 * o, a + 64 * o + 32 + 8 * kk, dhi + 2 * kk, idt, 1u);
            }
          } else {
#pragma unroll
            for (int k2 = 0; k2 < 2; ++k2) {
              const uint64_t b0 = interleave_kmajor_desc(bhi + k2 * 2 * 32 * 16, 32 * 16, 128);
              const uint64_t b1 = interleave_kmajor_desc(bhi + 2048 + k2 * 2 * 32 * 16, 32 * 16, 128);
              mma_f16_ts(dt + 32 * o, a + 32 * o + 8 * k2, b0, idb, k2 > 0 ? 1u : 0u);
              mma_f16_ts(dt + 32 * o, a + 32 * o + 8 * k2, b1, idb, 1u);
              mma_f16_ts(dt + 32 * o, a + 32 * o + 16 + 8 * k2, b0, idb, 1u);
            }
          }
        }
        for (int c = 0; c < ncommit; ++c) tc_commit(&cb[c]);
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    go = 1;
  } else if (side && warp < nside) {
    // columns [384, 512): disjoint from accumulators [0, 128) and A stages [128, 384)
    const uint32_t lb = tbase + ((uint32_t)((warp & 3) * 32) << 16) + 384 + 32 * ((warp >> 2) & 3);
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0x3f800000u + threadIdx.x + i;
    const int per = 32 / nside;  // st16 per warp per rep: 64 KB / 2 KB / nside
    while (!go) {
      for (int c = 0; c < per; ++c) {
        if (side == 1) {
          tmem_st16(lb + 16 * (c & 1), v);
        } else {
          tmem_ld16(lb + 16 * (c & 1), v);
        }
      }
      if (side == 1) {
        tc_wait_st();
      } else {
        tc_wait_ld_tied(v);
      }
    }
    if (v[2] == 777u) out[1000 + blockIdx.x] = v[1];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <bool BF>
void run(int side, int nside, int ncommit = 0) {
  unsigned long long* d;
  cudaMalloc(&d, 2000 * sizeof(unsigned long long));
  const int reps = 2000;
  mix<BF><<<148, 288>>>(50, side, nside, d, ncommit);
  mix<BF><<<148, 288>>>(reps, side, nside, d, ncommit);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  printf("%s side=%s x%d commits=%d: %7.1f cycles per block-pattern (%s)\n", BF ? "bf16x3 12 MMAs " : "3xtf32 24 MMAs ",
         side == 0 ? "none  " : side == 1 ? "stores" : "loads ", nside, ncommit, s / 148.0 / reps, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<false>(0, 0);
  run<false>(1, 4);
  run<false>(1, 8);
  run<false>(2, 4);
  run<true>(0, 0);
  run<true>(1, 4);
  run<true>(1, 8);
  run<true>(2, 4);
  run<false>(0, 0, 1);
  run<false>(0, 0, 3);
  run<false>(1, 8, 3);
  run<true>(0, 0, 3);
  return 0;
}
