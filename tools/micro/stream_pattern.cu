// Read bandwidth of a 4096 x 4096 fp64 row-major matrix by CTAs that own R rows x (n/S)
// columns and walk their columns in chunks of C doubles (C*8 contiguous bytes per row).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_pattern stream_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void walk(const double2* __restrict__ a, int n, int R, int S, int C, double* out) {
  const int rb = blockIdx.x / S, s = blockIdx.x % S;
  const int kper = n / S;
  const int pairs = C / 2;
  double acc = 0.0;
  for (int k0 = s * kper; k0 < (s + 1) * kper; k0 += C) {
    for (int i = threadIdx.x; i < R * pairs; i += blockDim.x) {
      const int r = i / pairs, c = i % pairs;
      double2 v = __ldg(a + ((size_t)(rb * R + r) * n + k0) / 2 + c);
      acc += v.x + v.y;
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  const int n = 4096;
  double2* a;
  double* out;
  cudaMalloc(&a, (size_t)n * n * 8);
  cudaMalloc(&out, 64);
  cudaMemset(a, 0, (size_t)n * n * 8);
  double* flush;
  cudaMalloc(&flush, 512 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int R : {16, 32, 64, 128})
    for (int C : {32, 64, 128, 256, 512}) {
      int S = 1;
      while ((n / R) * S < 296 && n / (2 * S) >= C) S *= 2;
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(flush, rep, 512 << 20);
        cudaEventRecord(e0);
        walk<<<(n / R) * S, 256>>>(a, n, R, S, C, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("R=%3d C=%3d (%4d B) S=%2d ctas=%4d: %6.1f us  %.2f TB/s\n", R, C, C * 8, S, (n / R) * S, best * 1e3,
             (double)n * n * 8 / (best * 1e-3) / 1e12);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
