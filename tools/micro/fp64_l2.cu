// Microbenchmarks for the DENSE-mode fp64 product design: DFMA and DMMA (m8n8k4) issue
// rates, and read bandwidth of an L2-sized working set re-read back to back.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_l2 fp64_l2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[4][2] = {};
  double af = threadIdx.x * 1e-3, bf = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[t][0]), "+d"(acc[t][1])
                   : "d"(af), "d"(bf));
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += acc[t][0] + acc[t][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int iters = 20000;
  dfma_kernel<<<148 * 8, 256>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  dfma_kernel<<<148 * 8, 256>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("DFMA: %.2f TFLOP/s\n", 2.0 * 148 * 8 * 256 * 8.0 * iters / (ms * 1e-3) / 1e12);
  dmma_kernel<<<148 * 8, 256>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  dmma_kernel<<<148 * 8, 256>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("DMMA m8n8k4: %.2f TFLOP/s\n", 2.0 * 148 * 8 * 8 * 4.0 * 256 * iters / (ms * 1e-3) / 1e12);
  for (size_t mb : {16, 32, 48, 64, 67, 80, 96, 110, 134, 256}) {
    size_t bytes = mb << 20;
    double2* p;
    cudaMalloc(&p, bytes);
    cudaMemset(p, 0, bytes);
    for (int grid : {148 * 4, 148 * 16}) {
      read_kernel<<<grid, 512>>>(p, bytes / 16, out);
      read_kernel<<<grid, 512>>>(p, bytes / 16, out);
      cudaEventRecord(a);
      const int reps = 20;
      for (int r = 0; r < reps; ++r) read_kernel<<<grid, 512>>>(p, bytes / 16, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("read %4zu MB grid %5d: %.2f TB/s (%.1f us per pass)\n", mb, grid, bytes * reps / (ms * 1e-3) / 1e12,
             ms * 1e3 / reps);
    }
    cudaFree(p);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
