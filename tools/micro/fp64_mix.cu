// Do DMMA (mma.sync m8n8k4 f64) and DFMA share the FP64 pipe on B200?  Times a loop of
// F independent DFMA chains per thread, M DMMAs per warp, and both in one loop body.
// Separate pipes: t(both) ~ max(t(dfma), t(dmma)); shared: t(both) ~ t(dfma) + t(dmma).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool DO_F, bool DO_M>
__global__ void mix_kernel(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  double acc[4][2] = {};
  const double b = 1.0000001, c = 1e-9;
  double af = threadIdx.x * 1e-3, bf = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
    if (DO_F) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    if (DO_M) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[t][0]), "+d"(acc[t][1])
                     : "d"(af), "d"(bf));
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  for (int t = 0; t < 4; ++t) s += acc[t][0] + acc[t][1];
  if (s == 12345.0) out[0] = s;
}

template <bool F, bool M>
float run(double* out, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  mix_kernel<F, M><<<148 * 8, 256>>>(out, 10);
  cudaEventRecord(a);
  mix_kernel<F, M><<<148 * 8, 256>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, 64);
  const int iters = 20000;
  const double thr = 148.0 * 8 * 256;
  float tf = run<true, false>(out, iters), tm = run<false, true>(out, iters), tb = run<true, true>(out, iters);
  const double ff = 2.0 * thr * 8 * iters, fm = 2.0 * (thr / 32) * 4 * 256 * iters;
  printf("DFMA only : %7.3f ms  %.2f TFLOP/s\n", tf, ff / (tf * 1e-3) / 1e12);
  printf("DMMA only : %7.3f ms  %.2f TFLOP/s\n", tm, fm / (tm * 1e-3) / 1e12);
  printf("both      : %7.3f ms  %.2f TFLOP/s total (sum of alone %.3f ms, max %.3f ms)\n", tb,
         (ff + fm) / (tb * 1e-3) / 1e12, tf + tm, tf > tm ? tf : tm);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
