// Tensor-pipe schedule of the fused operator, without the compute warps: how many cycles per
// 32-column block do the per-block MMAs + tcgen05.commit arrivals cost, by issue scheme?
//   A: two issuers (kernel r1): contraction warp 24 tf32 MMAs + 2 commits; distance warp 6 tf32
//      MMAs (no-swizzle B) + 2 commits
//   B: as A with the bf16x3 contraction (12 kind::f16 K=16 MMAs)
//   C: one issuer: distance 6 + contraction 24 (tf32) + 2 commits
//   D: one issuer: distance 6 + contraction 12 (bf16x3) + 2 commits
//   E: one issuer, two blocks per step: distance 6 N=64 + contraction 24 (bf16x3) + 2 commits
//   F: as D with 1 commit
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2503_02259_b200/csrc -o mma_sched mma_sched.cu
#include <cstdio>

#include "kgp_common.cuh"

using namespace kgp;

template <int MODE>
__global__ void sched(int reps, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sb[2 * 32 * 128];
  __shared__ __align__(1024) uint8_t sv[2 * 64 * 16 * 4];
  __shared__ uint64_t bar[2];
  __shared__ uint64_t cb[8];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 2 * 32 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3f803f80u;
  for (int i = threadIdx.x; i < 2 * 64 * 16; i += blockDim.x) reinterpret_cast<uint32_t*>(sv)[i] = 0x3f800000u;
  fence_proxy_async_smem();
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&cb[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  const uint32_t idt = idesc_tf32_m128(32), idb = idesc_bf16_m128(32), idd64 = idesc_tf32_m128(64);
  const uint32_t bhi = smem_u32(sb), va = smem_u32(sv);
  const uint64_t dhi = sw128_kmajor_desc(bhi), dlo = sw128_kmajor_desc(bhi + 32 * 128);
  // TMEM: accumulators [0, 128), distance [128, 192), U' [192, 224), A stages [256, 512)
  auto contraction = [&](int r) {
    const uint32_t dt = tbase + 64 * (r & 1);
    const uint32_t a = tbase + 256 + 128 * (r & 1);
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      if (MODE == 0 || MODE == 2 || MODE >= 6) {
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
  };
  auto distance = [&](int r, bool wide) {
    const uint32_t dd = tbase + 128 + (wide ? 0 : 32 * (r & 1));
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t uh = tbase + 192 + 8 * kk, ul = uh + 16;
      const int rows = wide ? 64 : 32;
      const uint64_t vh = interleave_kmajor_desc(va + kk * 2 * rows * 16, rows * 16, 128);
      const uint64_t vl = interleave_kmajor_desc(va + 4096 + kk * 2 * rows * 16, rows * 16, 128);
      const uint32_t id = wide ? idd64 : idt;
      mma_tf32_ts(dd, uh, vh, id, kk > 0 ? 1u : 0u);
      mma_tf32_ts(dd, uh, vl, id, 1u);
      mma_tf32_ts(dd, ul, vh, id, 1u);
    }
  };
  const long long t0 = clock64();
  if (MODE <= 1 || MODE >= 6) {
    if (warp == 8) {
      for (int r = 0; r < reps; ++r) {
        if (MODE == 6 || MODE == 7) {
          if (MODE == 7) mbar_wait(&cb[6], 1);  // a completed phase: returns at once
          tc_fence_after();
        }
        if (elect_one()) {
          contraction(r);
          tc_commit(&cb[0]);
          tc_commit(&cb[1]);
        }
        __syncwarp();
      }
      if (elect_one()) tc_commit(&bar[0]);
      __syncwarp();
      mbar_wait(&bar[0], 0);
      if ((threadIdx.x & 31) == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
    } else if (warp == 7) {
      for (int r = 0; r < reps; ++r) {
        if (elect_one()) {
          distance(r, false);
          tc_commit(&cb[2]);
          tc_commit(&cb[3]);
        }
        __syncwarp();
      }
      if (elect_one()) tc_commit(&bar[1]);
      __syncwarp();
      mbar_wait(&bar[1], 0);
      if ((threadIdx.x & 31) == 0) out[500 + blockIdx.x] = (unsigned long long)(clock64() - t0);
    }
  } else if (warp == 8) {
    const int steps = MODE == 4 ? reps / 2 : reps;
    for (int r = 0; r < steps; ++r) {
      if (elect_one()) {
        distance(r, MODE == 4);
        contraction(r);
        if (MODE == 4) contraction(r + 1);
        tc_commit(&cb[0]);
        if (MODE != 5) tc_commit(&cb[1]);
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar[0]);
    __syncwarp();
    mbar_wait(&bar[0], 0);
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int MODE>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 2000 * sizeof(unsigned long long));
  cudaMemset(d, 0, 2000 * sizeof(unsigned long long));
  const int reps = 2000;
  sched<MODE><<<148, 288>>>(50, d);
  sched<MODE><<<148, 288>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[1000];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)(h[i] > h[500 + i] ? h[i] : h[500 + i]);
  printf("%-62s %7.1f cycles per 32-column block (%s)\n", name, s / 148.0 / reps, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("A two issuers, tf32 24 + dist 6, 2+2 commits");
  run<1>("B two issuers, bf16x3 12 + dist 6, 2+2 commits");
  run<2>("C one issuer, dist 6 + tf32 24, 2 commits");
  run<3>("D one issuer, dist 6 + bf16x3 12, 2 commits");
  run<4>("E one issuer, 2 blocks/step: dist 6 (N=64) + bf16x3 24, 2 commits");
  run<5>("F one issuer, dist 6 + bf16x3 12, 1 commit");
  run<6>("G = A + tcgen05.fence::after_thread_sync per block (contraction warp)");
  run<7>("H = G + an mbarrier wait (completed phase) per block");
  return 0;
}
