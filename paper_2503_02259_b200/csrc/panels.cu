// Materialised rectangular panels and farthest-point sampling on the device.
//
// kgp_eval_panel replaces eval_kernel / eval_kernel_grad_l / pairwise_sq_dist
// (kernels.py:72-94) for the callers that need the panel itself: the landmark
// blocks K_mm, K_mn of the preconditioner build (precond.py:104-111) and the
// exact (dense) oracle path. kgp_fps replaces fps_select (precond.py:39-59).
#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

template <int KT>
__global__ void panel_kernel(int grad, int64_t nx, int64_t ny, int d, const double* __restrict__ x,
                             const double* __restrict__ y, double l, double* __restrict__ out, int64_t ldo) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = blockIdx.y;
  for (; i < nx; i += gridDim.y) {
    if (j >= ny) return;
    double acc = 0.0;  // direct differences, dimension order (_panels_numba.py:28-32)
    for (int q = 0; q < d; ++q) {
      double df = x[i * d + q] - y[j * d + q];
      acc = __dadd_rn(acc, __dmul_rn(df, df));  // no FMA contraction: numba's rounding
    }
    double v = grad == 2 ? acc : (grad == 1 ? dkappa64<KT>(acc, l) : kappa64<KT>(acc, l));
    out[i * ldo + j] = v;
  }
}

// numpy's pairwise summation order for a contiguous length-d reduction
// (np.sum(..., axis=1) in precond.py:53,58): sequential below 8 terms, eight
// interleaved partial sums combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) above.
__device__ inline double np_sqdist(const double* a, const double* b, int d) {
  if (d < 8) {
    double r = -0.0;
    for (int q = 0; q < d; ++q) {
      double t = a[q] - b[q];
      r = __dadd_rn(r, __dmul_rn(t, t));
    }
    return r;
  }
  double r[8];
  for (int q = 0; q < 8; ++q) {
    double t = a[q] - b[q];
    r[q] = __dmul_rn(t, t);
  }
  int q = 8;
  for (; q < d - (d % 8); q += 8)
    for (int u = 0; u < 8; ++u) {
      double t = a[q + u] - b[q + u];
      r[u] = __dadd_rn(r[u], __dmul_rn(t, t));
    }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; q < d; ++q) {
    double t = a[q] - b[q];
    res = __dadd_rn(res, __dmul_rn(t, t));
  }
  return res;
}

struct ArgMax {
  double v;
  int64_t i;
};
__device__ inline ArgMax better(ArgMax a, ArgMax b) {  // max value, lowest index on ties
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

// One FPS round: fold the point selected last round into the running minimum
// distances, then argmax. The last block to finish reduces the block partials
// (deterministic: the (value, index) order does not depend on arrival order).
__global__ void fps_round_kernel(int64_t n, int d, const double* __restrict__ x, double* __restrict__ dmin,
                                 int64_t* __restrict__ idx, int r, ArgMax* __restrict__ part,
                                 unsigned int* __restrict__ counter) {
  const int64_t p = idx[r - 1];
  double xp[16];
  for (int q = 0; q < d; ++q) xp[q] = x[p * d + q];
  ArgMax best{-1.0, INT64_MAX};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double dist = np_sqdist(x + i * d, xp, d);
    double v = (r == 1) ? dist : fmin(dmin[i], dist);
    dmin[i] = v;
    best = better(best, ArgMax{v, i});
  }
  __shared__ ArgMax sh[32];
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax other{__shfl_xor_sync(0xffffffffu, best.v, o), (int64_t)__shfl_xor_sync(0xffffffffu, best.i, o)};
    best = better(best, other);
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = better(best, sh[w]);
    part[blockIdx.x] = best;
    __threadfence();
    unsigned int done = atomicAdd(counter, 1u);
    if (done == gridDim.x - 1) {
      __threadfence();
      ArgMax g{__ldcg(&part[0].v), (int64_t)__ldcg((const long long*)&part[0].i)};
      for (unsigned int b = 1; b < gridDim.x; ++b)
        g = better(g, ArgMax{__ldcg(&part[b].v), (int64_t)__ldcg((const long long*)&part[b].i)});
      idx[r] = g.i;
      *counter = 0u;
    }
  }
}

__global__ void fps_seed_kernel(int64_t* idx, int64_t seed) { idx[0] = seed; }

}  // namespace

}  // namespace kgp

using namespace kgp;

extern "C" int kgp_eval_panel(int kernel, int grad, int64_t nx, int64_t ny, int d, const double* x, const double* y,
                              double l, double* out, int64_t ldo, void* stream) {
  KGP_REQUIRE(kernel >= 0 && kernel <= 2, KGP_ERR_INVALID, "unknown kernel id %d", kernel);
  KGP_REQUIRE(grad >= 0 && grad <= 2, KGP_ERR_INVALID, "grad selector must be 0, 1 or 2");
  KGP_REQUIRE(nx >= 0 && ny >= 0 && d >= 1 && ldo >= ny, KGP_ERR_INVALID, "bad panel shape");
  KGP_REQUIRE(l > 0.0, KGP_ERR_INVALID, "length scale must be positive and finite, got %g", l);
  if (nx == 0 || ny == 0) return KGP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)((ny + 127) / 128), (unsigned)(nx < 65535 ? nx : 65535));
  switch (kernel) {
    case GAUSS: panel_kernel<GAUSS><<<grid, 128, 0, st>>>(grad, nx, ny, d, x, y, l, out, ldo); break;
    case MAT32: panel_kernel<MAT32><<<grid, 128, 0, st>>>(grad, nx, ny, d, x, y, l, out, ldo); break;
    default: panel_kernel<MAT52><<<grid, 128, 0, st>>>(grad, nx, ny, d, x, y, l, out, ldo); break;
  }
  KGP_LAUNCH("panel_kernel");
  return KGP_OK;
}

extern "C" int kgp_fps(int64_t n, int d, const double* x, int64_t m, int64_t seed_index, int64_t* idx_out,
                       void* stream) {
  KGP_REQUIRE(n >= 1 && m >= 1 && m <= n, KGP_ERR_INVALID, "need 1 <= m <= n, got m=%lld, n=%lld", (long long)m,
              (long long)n);
  KGP_REQUIRE(seed_index >= 0 && seed_index < n, KGP_ERR_INVALID, "seed_index %lld out of range for n=%lld",
              (long long)seed_index, (long long)n);
  KGP_REQUIRE(d >= 1 && d <= 16, KGP_ERR_INVALID, "fps supports 1 <= d <= 16");
  cudaStream_t st = (cudaStream_t)stream;
  fps_seed_kernel<<<1, 1, 0, st>>>(idx_out, seed_index);
  KGP_LAUNCH("fps_seed_kernel");
  if (m == 1) return KGP_OK;
  int nb = (int)((n + 255) / 256);
  if (nb > 296) nb = 296;  // 2 waves of 148 SMs
  DevBuf scratch;
  size_t bytes = sizeof(double) * n + sizeof(ArgMax) * nb + 16;
  int rc = scratch.ensure(bytes);
  if (rc) return rc;
  double* dmin = scratch.as<double>();
  ArgMax* part = reinterpret_cast<ArgMax*>(dmin + n);
  unsigned int* counter = reinterpret_cast<unsigned int*>(part + nb);
  KGP_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned int), st));
  for (int64_t r = 1; r < m; ++r) {
    fps_round_kernel<<<nb, 256, 0, st>>>(n, d, x, dmin, idx_out, (int)r, part, counter);
    KGP_LAUNCH("fps_round_kernel");
  }
  KGP_CUDA(cudaStreamSynchronize(st));  // scratch is released on return
  return KGP_OK;
}
