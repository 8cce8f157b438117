// TMEM traffic microbenchmarks (one CTA per SM, 148 CTAs): is the fused operator's
// A-tile store stream (tcgen05.st) or its interaction with the contraction MMAs the
// per-block bound? Measures, in cycles at 1965 MHz:
//   st:   NW warps storing 32x32b.x16 (2 KB per warp-instruction), bytes/cycle/SM
//   ld:   NW warps loading 32x32b.x16 + wait::ld
//   mma:  tf32 M=128 N=32 K=8 (A in TMEM) and bf16 kind::f16 M=128 N=32 K=16 (A in TMEM)
//   mix:  stores and tf32 MMAs concurrently (different TMEM columns): overlapped or serial?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2503_02259_b200/csrc -o tmem_bw tmem_bw.cu
#include <cstdio>

#include "kgp_common.cuh"

using namespace kgp;

// mode: 0 st only, 1 ld only, 2 tf32 mma only, 3 bf16 mma only, 4 st + tf32 mma, 5 st + bf16 mma
template <int MODE>
__global__ void tmem_bench(int reps, int nst_warps, int mma_per_rep, unsigned long long* cyc_out) {
  __shared__ __align__(1024) uint8_t sb[32 * 128 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 32 * 128 * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3f803f80u;
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
  const long long t0 = clock64();
  const int mma_warp = 8;
  if ((MODE == 0 || MODE == 1 || MODE >= 4) && warp < nst_warps) {
    // warp w: lane quadrant w%4, columns [128 + 64 * (w/4), +64) cycled in 16-column steps
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16) + 128 + 64 * (warp >> 2);
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0x3f800000u + threadIdx.x + i;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (MODE == 1) {
          tmem_ld16(lane_base + 16 * c, v);
        } else {
          tmem_st16(lane_base + 16 * c, v);
        }
      }
      if (MODE == 1) {
        tc_wait_ld_tied(v);
        v[0] += 1;
      }
    }
    if (MODE == 1) {
      tc_wait_ld();
    } else {
      tc_wait_st();
    }
    if (v[3] == 12345u) cyc_out[blockIdx.x + 1000] = v[5];
  }
  if (MODE >= 2 && warp == mma_warp) {
    const uint32_t idt = idesc_tf32_m128(32);
    const uint32_t idb = idesc_bf16_m128(32);
    const uint64_t bd = sw128_kmajor_desc(smem_u32(sb));
    const uint64_t bi = interleave_kmajor_desc(smem_u32(sb), 32 * 16, 128);
    for (int r = 0; r < reps; ++r) {
      if (elect_one()) {
        for (int kk = 0; kk < mma_per_rep; ++kk) {
          if (MODE == 2 || MODE == 4)
            mma_tf32_ts(tbase + 32 * (kk & 1), tbase + 384 + 8 * (kk & 3), bd + 2 * (kk & 3), idt, 1u);
          else
            mma_f16_ts(tbase + 32 * (kk & 1), tbase + 384 + 8 * (kk & 3), bi, idb, 1u);
        }
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long tm = clock64();
    if ((threadIdx.x & 31) == 0) cyc_out[blockIdx.x + 500] = (unsigned long long)(tm - t0);
  }
  tc_fence_before();
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc_out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int MODE>
double run(int reps, int nst, int mpr) {
  unsigned long long* d;
  cudaMalloc(&d, 2000 * sizeof(unsigned long long));
  cudaMemset(d, 0, 2000 * sizeof(unsigned long long));
  tmem_bench<MODE><<<148, 384>>>(4, nst, mpr, d);
  tmem_bench<MODE><<<148, 384>>>(reps, nst, mpr, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) printf("mode %d: %s\n", MODE, cudaGetErrorString(e));
  unsigned long long h[1000];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  double s = 0, sm = 0;
  for (int i = 0; i < 148; ++i) {
    s += (double)h[i];
    sm += (double)h[500 + i];
  }
  if (MODE >= 2) printf("   (mode %d: block %.1f, mma warp %.1f cycles/rep)\n", MODE, s / 148.0 / reps, sm / 148.0 / reps);
  return s / 148.0 / reps;  // cycles per rep
}

int main() {
  const int reps = 4000;
  for (int nst : {4, 8, 12}) {
    double c = run<0>(reps, nst, 0);
    printf("st  %2d warps: %7.1f cycles/rep, %6.1f B/cycle (each rep: %d x 4 x 2 KB)\n", nst, c,
           nst * 4 * 2048.0 / c, nst);
    c = run<1>(reps, nst, 0);
    printf("ld  %2d warps: %7.1f cycles/rep, %6.1f B/cycle\n", nst, c, nst * 4 * 2048.0 / c);
  }
  for (int mpr : {4, 8}) {
    double c = run<2>(reps, 0, mpr);
    printf("tf32 mma N=32 K=8 : %6.2f cycles/MMA\n", c / mpr);
    c = run<3>(reps, 0, mpr);
    printf("bf16 mma N=32 K=16: %6.2f cycles/MMA\n", c / mpr);
  }
  // concurrent: 8 store warps (16 KB / rep) + tf32 MMAs
  for (int mpr : {4, 8, 12}) {
    const double cs = run<0>(reps, 8, 0), cm = run<2>(reps, 0, mpr), cx = run<4>(reps, 8, mpr);
    printf("mix st(8w x 8 KB) + %2d tf32 MMAs: st alone %7.1f, mma alone %7.1f, both %7.1f cycles/rep\n", mpr, cs,
           cm, cx);
    const double cb = run<3>(reps, 0, mpr), cy = run<5>(reps, 8, mpr);
    printf("mix st(8w x 8 KB) + %2d bf16 MMAs: st alone %7.1f, mma alone %7.1f, both %7.1f cycles/rep\n", mpr, cs,
           cb, cy);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
