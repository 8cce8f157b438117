// Streaming read bandwidth of 1-D cp.async.bulk copies (size S per copy, L copies per
// stage, 4-stage ring, consumer warps only release the stage) over a 134 MB matrix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2503_02259_b200/csrc -o bulk_stream bulk_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("{.reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0];}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}" ::"r"(
                   su32(b)),
               "r"(par)
               : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(d)),
               "l"(s), "r"(bytes), "r"(su32(b))
               : "memory");
}

// CTA streams `per_cta` bytes starting at base + blockIdx.x * per_cta, as lines of S bytes
// taken from rows of `rowbytes` (line i of stage c: row (c*L + i) % rows... simple: contiguous)
__global__ void stream(const char* base, size_t per_cta, int S, int L, int stages, int rowstride_mode) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], cw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t stage_bytes = (size_t)S * L;
  const int nchunks = (int)(per_cta / stage_bytes);
  const char* src = base + blockIdx.x * per_cta;
  if (warp == cw) {
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % stages;
      if (c >= stages) wait(&empty[s], ((c / stages) - 1) & 1);
      if (lane == 0) arrive_tx(&full[s], (uint32_t)stage_bytes);
      __syncwarp();
      for (int i = lane; i < L; i += 32) {
        // rowstride_mode 1: line i comes from a different 32 KB "row" (matrix-like access)
        const char* p = rowstride_mode ? src + (size_t)i * (per_cta / L) + (size_t)c * S : src + (size_t)c * stage_bytes + (size_t)i * S;
        bulk(sm + s * stage_bytes + (size_t)i * S, p, S, &full[s]);
      }
    }
  } else {
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % stages;
      wait(&full[s], (c / stages) & 1);
      __syncwarp();
      if (lane == 0) arrive(&empty[s]);
    }
  }
}

int main() {
  const size_t total = 134217728;
  char* a;
  cudaMalloc(&a, total);
  cudaMemset(a, 1, total);
  char* fl;
  cudaMalloc(&fl, 512 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode)
    for (int S : {256, 512, 1024, 2048, 4096})
      for (int ctas : {128, 148, 296}) {
        const int stages = 4;
        const int L = 49152 / S;  // 48 KB per stage
        const size_t smem = (size_t)stages * S * L;
        if (ctas == 296 && smem > 110 * 1024) continue;
        const size_t per = total / ctas / (S * L) * (S * L);
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
          cudaMemset(fl, r, 512 << 20);
          cudaEventRecord(e0);
          stream<<<ctas, 288, smem>>>(a, per, S, L, stages, mode);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          best = ms < best ? ms : best;
        }
        printf("mode %d S=%5d L=%3d ctas=%3d: %.2f TB/s\n", mode, S, L, ctas, per * ctas / (best * 1e-3) / 1e12);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
