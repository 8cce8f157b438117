// tcgen05.mma kind::tf32 throughput vs N (M=128, K=8 per instruction), A from TMEM (ts)
// or shared memory (ss), B from shared memory: is a 128x32x8 MMA (the fused operator's
// contraction shape at k=32) as efficient per flop as a wide one?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2503_02259_b200/csrc -o mma_n mma_n.cu
#include <cstdio>

#include "kgp_common.cuh"

using namespace kgp;

template <int N, bool TS>
__global__ void mma_rate(int reps) {
  __shared__ __align__(1024) uint8_t sb[224 * 128];
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 224 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3f800000u;
  for (int i = threadIdx.x; i < 128 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sa)[i] = 0x3f800000u;
  fence_proxy_async_smem();
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (warp == 0) {
    const uint32_t idesc = idesc_tf32_m128(N);
    const uint64_t bd = sw128_kmajor_desc(smem_u32(sb));
    const uint64_t ad = sw128_kmajor_desc(smem_u32(sa));
    for (int r = 0; r < reps; ++r) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (TS)
            mma_tf32_ts(tbase, tbase + 256 + 8 * kk, bd + 2 * kk, idesc, 1u);
          else
            mma_tf32_ss(tbase, ad + 2 * kk, bd + 2 * kk, idesc, 1u);
        }
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int N, bool TS>
void run(int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  mma_rate<N, TS><<<148, 128>>>(10);
  cudaEventRecord(a);
  mma_rate<N, TS><<<148, 128>>>(reps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fl = 148.0 * reps * 4 * 2.0 * 128 * N * 8;
  const double cyc = ms * 1e-3 * 1.965e9 / (reps * 4.0);
  printf("N=%3d %s: %7.1f TFLOP/s  %6.2f cycles per MMA (at 1965 MHz)\n", N, TS ? "ts" : "ss", fl / (ms * 1e-3) / 1e12,
         cyc);
}

int main() {
  const int reps = 20000;
  run<32, true>(reps);
  run<64, true>(reps);
  run<128, true>(reps);
  run<224, true>(reps);
  run<32, false>(reps);
  run<64, false>(reps);
  run<128, false>(reps);
  run<224, false>(reps);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
