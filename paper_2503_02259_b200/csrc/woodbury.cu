// Woodbury application of the landmark preconditioner on the device.
//
// NystromPreconditioner.apply_inverse (precond.py:74-83) computes
//   out = B / s - V cho_solve(C, V^T B) / s^2,   C = I/f^2 + V^T V / s.
// With C = L_C L_C^T factored once at build time and W = V L_C^-T, this is
//   out = B / s - W (W^T B) / s^2
// two tall-skinny fp64 GEMMs per application and no triangular solve in the
// PCG loop. Both GEMMs run on one tiled fp64 kernel (64x64 tiles, split-K with
// a fixed-order partial reduction so results are run-to-run deterministic).
#include <cublas_v2.h>
#include <stdlib.h>

#include <map>

#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

// One cuBLAS handle per (host thread, device): a handle must not be used by two threads at
// once, and the callers are stream-ordered on the stream passed in.
static int cublas_for_device(cublasHandle_t* out) {
  thread_local std::map<int, cublasHandle_t> handles;
  int dev = 0;
  KGP_CUDA(cudaGetDevice(&dev));
  auto it = handles.find(dev);
  if (it == handles.end()) {
    cublasHandle_t h;
    KGP_REQUIRE(cublasCreate(&h) == CUBLAS_STATUS_SUCCESS, KGP_ERR_CUDA, "cublasCreate failed");
    it = handles.emplace(dev, h).first;
  }
  *out = it->second;
  return KGP_OK;
}

// C = alpha op(A) op(B) + beta SRC through cublasDgemm when every operand has a unit stride
// along one index and C is column-major (c_is == 1). Returns 1 when the layout does not fit.
static int gemm_f64_cublas(int64_t M, int64_t N, int64_t K, const double* a, int64_t a_is, int64_t a_ks,
                           const double* b, int64_t b_ks, int64_t b_ns, double* c, int64_t c_ns, double alpha,
                           double beta, const double* src, int64_t s_is, int64_t s_ns, cudaStream_t st) {
  const bool a_n = (a_is == 1), a_t = (a_ks == 1);
  const bool b_n = (b_ks == 1), b_t = (b_ns == 1);
  if (!(a_n || a_t) || !(b_n || b_t) || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return 1;
  if (beta != 0.0 && src != c) {
    if (src == nullptr || s_is != 1) return 1;
    KGP_CUDA(cudaMemcpy2DAsync(c, sizeof(double) * c_ns, src, sizeof(double) * s_ns, sizeof(double) * M, N,
                               cudaMemcpyDeviceToDevice, st));
  }
  cublasHandle_t h;
  int rc = cublas_for_device(&h);
  if (rc) return rc;
  KGP_REQUIRE(cublasSetStream(h, st) == CUBLAS_STATUS_SUCCESS, KGP_ERR_CUDA, "cublasSetStream failed");
  const cublasStatus_t cs =
      cublasDgemm(h, a_n ? CUBLAS_OP_N : CUBLAS_OP_T, b_n ? CUBLAS_OP_N : CUBLAS_OP_T, (int)M, (int)N, (int)K, &alpha, a,
                  (int)(a_n ? (a_ks > 1 ? a_ks : M) : (a_is > 1 ? a_is : K)), b,
                  (int)(b_n ? (b_ns > 1 ? b_ns : K) : (b_ks > 1 ? b_ks : N)), &beta, c, (int)(c_ns > 1 ? c_ns : M));
  KGP_REQUIRE(cs == CUBLAS_STATUS_SUCCESS, KGP_ERR_CUDA, "cublasDgemm failed (%d)", (int)cs);
  count_launches(1);
  return KGP_OK;
}

namespace {

constexpr int BM = 64, BN = 64, BK = 16, GT = 256;

struct GemmArgs {
  int64_t M, N, K;             // C (M x N) = A (M x K) . B (K x N)
  const double* a;
  int64_t a_is, a_ks;          // A(i, q) = a[i*a_is + q*a_ks]
  const double* b;
  int64_t b_ks, b_ns;          // B(q, c) = b[q*b_ks + c*b_ns]
  double* c;                   // partial or final output
  int64_t c_is, c_ns;
  int64_t kchunk;              // split-K chunk (grid.z slices)
  int64_t part_stride;         // elements between split-K partial slices (0: final)
  double alpha, beta;          // final: c = beta * src + alpha * acc
  const double* src;
  int64_t s_is, s_ns;
};

__global__ void __launch_bounds__(GT) dgemm_kernel(const GemmArgs g) {
  __shared__ double As[BK][BM + 1];
  __shared__ double Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = (int64_t)blockIdx.x * BM, c0 = (int64_t)blockIdx.y * BN;
  const int64_t q_begin = (int64_t)blockIdx.z * g.kchunk;
  const int64_t q_end = q_begin + g.kchunk < g.K ? q_begin + g.kchunk : g.K;
  double acc[4][4] = {};
  const bool a_i_contig = (g.a_is == 1);
  const bool b_n_contig = (g.b_ns == 1);
  for (int64_t q0 = q_begin; q0 < q_end; q0 += BK) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      int e = tid + GT * t;
      int ii, qq;
      if (a_i_contig) { ii = e % BM; qq = e / BM; } else { qq = e % BK; ii = e / BK; }
      int64_t gi = i0 + ii, gq = q0 + qq;
      As[qq][ii] = (gi < g.M && gq < q_end) ? g.a[gi * g.a_is + gq * g.a_ks] : 0.0;
      int cc;
      if (b_n_contig) { cc = e % BN; qq = e / BN; } else { qq = e % BK; cc = e / BK; }
      int64_t gc = c0 + cc;
      gq = q0 + qq;
      Bs[qq][cc] = (gc < g.N && gq < q_end) ? g.b[gq * g.b_ks + gc * g.b_ns] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int qq = 0; qq < BK; ++qq) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = As[qq][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = Bs[qq][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int64_t gi = i0 + ty + 16 * u, gc = c0 + tx + 16 * v;
      if (gi >= g.M || gc >= g.N) continue;
      if (g.part_stride) {
        g.c[blockIdx.z * g.part_stride + gi * g.c_is + gc * g.c_ns] = acc[u][v];
      } else {
        double val = g.alpha * acc[u][v];
        if (g.src) val += g.beta * g.src[gi * g.s_is + gc * g.s_ns];
        g.c[gi * g.c_is + gc * g.c_ns] = val;
      }
    }
}

// c[e] = sum_z part[z * stride + e], fixed order in z
__global__ void sum_partials_kernel(int64_t count, int nz, int64_t stride, const double* __restrict__ part,
                                    double* __restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  double s = 0.0;
  for (int z = 0; z < nz; ++z) s += part[z * stride + e];
  out[e] = s;
}

// c[i, j] = alpha * sum_z part[z][i, j] + beta * src[i, j], fixed order in z
__global__ void finish_partials_kernel(int64_t M, int64_t N, int nz, const double* __restrict__ part, double alpha,
                                       double beta, const double* __restrict__ src, int64_t s_is, int64_t s_ns,
                                       double* __restrict__ c, int64_t c_is, int64_t c_ns) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const int64_t i = e / N, j = e % N;
  double acc = 0.0;
  for (int z = 0; z < nz; ++z) acc += part[(int64_t)z * M * N + e];
  double v = alpha * acc;
  if (src) v += beta * src[i * s_is + j * s_ns];
  c[i * c_is + j * c_ns] = v;
}

// ------------------------------------------------------------------ skinny products (N <= 8 RHS)
// The 64x64-tile kernel wastes 63/64 of its work and most of the machine when N is 1..8
// (the PCG w-solve applies M^-1 to ONE column every iteration). These two kernels are
// plain HBM/L2 streams over A with the N right-hand-side values broadcast, each writing
// fixed-order split-K partials (deterministic) finished by finish_partials_kernel.
constexpr int SK_MAXN = 8;

// single K chunk: the kernels write C = alpha acc + beta SRC themselves (no partials pass)
struct SkEpi {
  double alpha, beta;
  const double* src;
  int64_t s_is, s_ns;
  double* c;
  int64_t c_is, c_ns;
  KGP_DEV void put(double* part, int64_t M, int N, int64_t i, int col, double v) const {
    if (gridDim.y == 1) {
      double o = alpha * v;
      if (src) o += beta * src[i * s_is + col * s_ns];
      c[i * c_is + col * c_ns] = o;
    } else {
      part[((int64_t)blockIdx.y * M + i) * N + col] = v;
    }
  }
};

// A rows contiguous along K (a_ks == 1): one CTA per (output row, K chunk); threads stride
// the chunk with four independent loads in flight each, block-reduced in fixed order.
template <int N>
__global__ void __launch_bounds__(256) skinny_rowdot_kernel(int64_t M, int64_t K, int64_t kchunk,
                                                            const double* __restrict__ a, int64_t a_is,
                                                            const double* __restrict__ b, int64_t b_ks, int64_t b_ns,
                                                            double* __restrict__ part, SkEpi epi) {
  const int64_t i = blockIdx.x;
  const int64_t q0 = (int64_t)blockIdx.y * kchunk;
  const int64_t q1 = q0 + kchunk < K ? q0 + kchunk : K;
  const double* ar = a + i * a_is;
  double acc[4][N];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int c = 0; c < N; ++c) acc[u][c] = 0.0;
  int64_t q = q0 + threadIdx.x;
  for (; q + 3 * 256 < q1; q += 4 * 256) {
    double av[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) av[u] = ar[q + u * 256];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < N; ++c) acc[u][c] = fma(av[u], b[(q + u * 256) * b_ks + c * b_ns], acc[u][c]);
  }
  for (; q < q1; q += 256)
#pragma unroll
    for (int c = 0; c < N; ++c) acc[0][c] = fma(ar[q], b[q * b_ks + c * b_ns], acc[0][c]);
  __shared__ double red[8][N];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    const double v = warp_sum((acc[0][c] + acc[1][c]) + (acc[2][c] + acc[3][c]));
    if (lane == 0) red[w][c] = v;
  }
  __syncthreads();
  if (threadIdx.x < N) {
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v += red[k][threadIdx.x];
    epi.put(part, M, N, i, threadIdx.x, v);
  }
}

// short rows (K chunk < 4096): one warp per output row, lanes stride K, 4 loads in flight
template <int N>
__global__ void __launch_bounds__(256) skinny_rowwarp_kernel(int64_t M, int64_t K, const double* __restrict__ a,
                                                             int64_t a_is, const double* __restrict__ b,
                                                             int64_t b_ks, int64_t b_ns, double* __restrict__ part,
                                                             SkEpi epi) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= M) return;
  const double* ar = a + i * a_is;
  double acc[4][N];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int c = 0; c < N; ++c) acc[u][c] = 0.0;
  int64_t q = lane;
  for (; q + 96 < K; q += 128) {
    double av[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) av[u] = ar[q + 32 * u];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < N; ++c) acc[u][c] = fma(av[u], b[(q + 32 * u) * b_ks + c * b_ns], acc[u][c]);
  }
  for (; q < K; q += 32)
#pragma unroll
    for (int c = 0; c < N; ++c) acc[0][c] = fma(ar[q], b[q * b_ks + c * b_ns], acc[0][c]);
#pragma unroll
  for (int c = 0; c < N; ++c) {
    const double v = warp_sum((acc[0][c] + acc[1][c]) + (acc[2][c] + acc[3][c]));
    if (lane == 0) epi.put(part, M, N, i, c, v);
  }
}

// A contiguous along M (a_is == 1): one thread per output row, the B chunk staged in smem.
constexpr int SK_QC = 128;
template <int N>
__global__ void __launch_bounds__(256) skinny_col_kernel(int64_t M, int64_t K, int64_t kchunk,
                                                         const double* __restrict__ a, int64_t a_ks,
                                                         const double* __restrict__ b, int64_t b_ks, int64_t b_ns,
                                                         double* __restrict__ part, SkEpi epi) {
  __shared__ double bs[SK_QC * N];
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t q0 = (int64_t)blockIdx.y * kchunk;
  const int64_t q1 = q0 + kchunk < K ? q0 + kchunk : K;
  double acc[N];
#pragma unroll
  for (int c = 0; c < N; ++c) acc[c] = 0.0;
  for (int64_t qb = q0; qb < q1; qb += SK_QC) {
    const int nq = (int)(q1 - qb < SK_QC ? q1 - qb : SK_QC);
    __syncthreads();
    for (int e = threadIdx.x; e < nq * N; e += 256) bs[e] = b[(qb + e / N) * b_ks + (e % N) * b_ns];
    __syncthreads();
    if (i < M) {
      const double* ac = a + i + qb * a_ks;
      int q = 0;
      for (; q + 8 <= nq; q += 8) {
        double av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) av[u] = ac[(int64_t)(q + u) * a_ks];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int c = 0; c < N; ++c) acc[c] = fma(av[u], bs[(q + u) * N + c], acc[c]);
      }
      for (; q < nq; ++q)
#pragma unroll
        for (int c = 0; c < N; ++c) acc[c] = fma(ac[(int64_t)q * a_ks], bs[q * N + c], acc[c]);
    }
  }
  if (i >= M) return;
#pragma unroll
  for (int c = 0; c < N; ++c) epi.put(part, M, N, i, c, acc[c]);
}

template <int N>
int skinny_launch(int kind, int64_t M, int64_t K, int64_t nz, int64_t kchunk, const double* a, int64_t a_is,
                  int64_t a_ks, const double* b, int64_t b_ks, int64_t b_ns, double* part, const SkEpi& epi,
                  cudaStream_t st) {
  if (kind == 2) {
    skinny_rowwarp_kernel<N><<<(unsigned)((M + 7) / 8), 256, 0, st>>>(M, K, a, a_is, b, b_ks, b_ns, part, epi);
    KGP_LAUNCH("skinny_rowwarp_kernel");
  } else if (kind == 1) {
    skinny_rowdot_kernel<N><<<dim3((unsigned)M, (unsigned)nz), 256, 0, st>>>(M, K, kchunk, a, a_is, b, b_ks, b_ns,
                                                                             part, epi);
    KGP_LAUNCH("skinny_rowdot_kernel");
  } else {
    skinny_col_kernel<N><<<dim3((unsigned)((M + 255) / 256), (unsigned)nz), 256, 0, st>>>(M, K, kchunk, a, a_ks, b,
                                                                                          b_ks, b_ns, part, epi);
    KGP_LAUNCH("skinny_col_kernel");
  }
  return KGP_OK;
}

// C = alpha A B + beta SRC for N <= SK_MAXN; A has a unit stride along K or along M
int skinny_gemm(int64_t M, int64_t N, int64_t K, const double* a, int64_t a_is, int64_t a_ks, const double* b,
                int64_t b_ks, int64_t b_ns, double* c, int64_t c_is, int64_t c_ns, double alpha, double beta,
                const double* src, int64_t s_is, int64_t s_ns, DevBuf& tmp, cudaStream_t st) {
  // kind 1: CTA per (row, K chunk) for long rows; 2: warp per row for short rows; 0: column kernel
  // (a warp per row only when there are enough rows to fill the machine with warps and the
  // rows are short; otherwise CTAs stream row chunks)
  const int kind = (a_ks == 1) ? ((K < 8192 && M >= 4096) ? 2 : 1) : 0;
  int64_t nz = 1, kchunk = K > 0 ? K : 1;
  if (kind != 2) {
    const int64_t gx = kind == 1 ? M : (M + 255) / 256;
    // K chunks: enough CTAs for ~8 per SM, each streaming >= 1024 (row) / 32 (column) elements
    // short rows: one CTA per row writes C directly (no partials pass); long rows / few
    // rows: K chunks for memory-level parallelism
    nz = (kind == 1 && K <= 8192) ? 1 : (1184 + gx - 1) / gx;
    const int64_t min_chunk = kind == 1 ? 1024 : 32;
    if (nz > (K + min_chunk - 1) / min_chunk) nz = (K + min_chunk - 1) / min_chunk;
    if (nz < 1) nz = 1;
    if (nz > 65535) nz = 65535;
    kchunk = (K + nz - 1) / nz;
    if (kchunk < 1) kchunk = 1;
    nz = (K + kchunk - 1) / kchunk;
    if (nz < 1) nz = 1;
  }
  int rc = tmp.ensure(sizeof(double) * (size_t)(M * N * nz));
  if (rc) return rc;
  double* part = tmp.as<double>();
  const SkEpi epi{alpha, beta, src, s_is, s_ns, c, c_is, c_ns};
  const bool direct = K > 0 && (kind == 2 || nz == 1);  // the kernel writes C itself
  if (K <= 0) {
    KGP_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * M * N, st));
  } else {
    switch (N) {
#define KGP_SK(NN) \
  case NN: rc = skinny_launch<NN>(kind, M, K, nz, kchunk, a, a_is, a_ks, b, b_ks, b_ns, part, epi, st); break;
      KGP_SK(1) KGP_SK(2) KGP_SK(3) KGP_SK(4) KGP_SK(5) KGP_SK(6) KGP_SK(7) KGP_SK(8)
#undef KGP_SK
    }
    if (rc) return rc;
  }
  if (direct) return KGP_OK;
  finish_partials_kernel<<<(unsigned)((M * N + 255) / 256), 256, 0, st>>>(M, N, (int)nz, part, alpha, beta, src,
                                                                          s_is, s_ns, c, c_is, c_ns);
  KGP_LAUNCH("finish_partials_kernel");
  return KGP_OK;
}

}  // namespace

int gemm_f64(int64_t M, int64_t N, int64_t K, const double* a, int64_t a_is, int64_t a_ks, const double* b,
             int64_t b_ks, int64_t b_ns, double* c, int64_t c_is, int64_t c_ns, double alpha, double beta,
             const double* src, int64_t s_is, int64_t s_ns, DevBuf& tmp, cudaStream_t st) {
  if (M <= 0 || N <= 0) return KGP_OK;
  if (N <= SK_MAXN && (a_ks == 1 || a_is == 1))
    return skinny_gemm(M, N, K, a, a_is, a_ks, b, b_ks, b_ns, c, c_is, c_ns, alpha, beta, src, s_is, s_ns, tmp, st);
  // wider right-hand-side blocks: cuBLAS DGEMM (a plain library GEMM, DMMA; the tiled SIMT
  // kernel below stays for layouts it cannot express). Env KGP_GEMM_CUBLAS=0 disables it.
  static const bool use_cublas = [] {
    const char* e = getenv("KGP_GEMM_CUBLAS");
    return !(e && atoi(e) == 0);
  }();
  if (use_cublas && c_is == 1) {
    const int rc = gemm_f64_cublas(M, N, K, a, a_is, a_ks, b, b_ks, b_ns, c, c_ns, alpha, beta, src, s_is, s_ns, st);
    if (rc != 1) return rc;
  }
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int64_t nz = 1;
  if (tiles < 148 && K > 4096) {  // too few output tiles to fill the SMs: split K, fixed-order reduction
    nz = (K + 2047) / 2048;
    int64_t cap = 296 / tiles;
    if (cap < 1) cap = 1;
    if (nz > cap) nz = cap;
  }
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.a = a; g.a_is = a_is; g.a_ks = a_ks;
  g.b = b; g.b_ks = b_ks; g.b_ns = b_ns;
  if (nz <= 1) {
    g.c = c; g.c_is = c_is; g.c_ns = c_ns;
    g.kchunk = K > 0 ? K : 1; g.part_stride = 0;
    g.alpha = alpha; g.beta = beta;
    g.src = src; g.s_is = s_is; g.s_ns = s_ns;
    dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), 1);
    dgemm_kernel<<<grid, GT, 0, st>>>(g);
    KGP_LAUNCH("dgemm_kernel");
    return KGP_OK;
  }
  const int64_t kchunk = ((K + nz - 1) / nz + BK - 1) / BK * BK;
  nz = (K + kchunk - 1) / kchunk;
  int rc = tmp.ensure(sizeof(double) * (size_t)(M * N * nz));
  if (rc) return rc;
  g.c = tmp.as<double>(); g.c_is = N; g.c_ns = 1;
  g.kchunk = kchunk; g.part_stride = M * N;
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), (unsigned)nz);
  dgemm_kernel<<<grid, GT, 0, st>>>(g);
  KGP_LAUNCH("dgemm_kernel (split-K)");
  finish_partials_kernel<<<(unsigned)((M * N + 255) / 256), 256, 0, st>>>(M, N, (int)nz, tmp.as<double>(), alpha,
                                                                            beta, src, s_is, s_ns, c, c_is, c_ns);
  KGP_LAUNCH("finish_partials_kernel");
  return KGP_OK;
}

// T = U^T B (m x k, row-major), U^T = p->wt (m x n); split over n with fixed-order partials
int lowrank_project_impl(kgp_precond_s* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* T,
                         cudaStream_t st) {
  const int64_t n = p->n, m = p->m;
  if (k <= SK_MAXN)
    return skinny_gemm(m, k, n, p->wt.as<double>(), n, 1, b, b_rs, b_cs, T, k, 1, 1.0, 0.0, nullptr, 0, 0, p->tmp, st);
  int64_t tiles = ((m + BM - 1) / BM) * ((k + BN - 1) / BN);
  int64_t nz = (n + 2047) / 2048;
  int64_t cap = 296 / tiles;
  if (cap < 1) cap = 1;
  if (nz > cap) nz = cap;
  int64_t kchunk = ((n + nz - 1) / nz + BK - 1) / BK * BK;
  nz = (n + kchunk - 1) / kchunk;
  int rc = p->tmp.ensure(sizeof(double) * (size_t)m * k * nz);
  if (rc) return rc;
  double* part = p->tmp.as<double>();
  GemmArgs g{};
  g.M = m; g.N = k; g.K = n;
  g.a = p->wt.as<double>(); g.a_is = n; g.a_ks = 1;
  g.b = b; g.b_ks = b_rs; g.b_ns = b_cs;
  g.c = part; g.c_is = k; g.c_ns = 1;
  g.kchunk = kchunk; g.part_stride = m * k;
  dim3 grid1((unsigned)((m + BM - 1) / BM), (unsigned)((k + BN - 1) / BN), (unsigned)nz);
  dgemm_kernel<<<grid1, GT, 0, st>>>(g);
  KGP_LAUNCH("dgemm_kernel (U^T B)");
  sum_partials_kernel<<<(unsigned)((m * k + 255) / 256), 256, 0, st>>>(m * k, (int)nz, m * k, part, T);
  KGP_LAUNCH("sum_partials_kernel");
  return KGP_OK;
}

// out = beta B + alpha U T
int lowrank_expand_impl(kgp_precond_s* p, double beta, double alpha, int64_t k, const double* b, int64_t b_rs,
                        int64_t b_cs, const double* T, double* out, int64_t o_rs, int64_t o_cs, cudaStream_t st) {
  const int64_t n = p->n, m = p->m;
  if (k <= SK_MAXN)
    return skinny_gemm(n, k, m, p->wt.as<double>(), 1, n, T, k, 1, out, o_rs, o_cs, alpha, beta, b, b_rs, b_cs,
                       p->tmp2, st);
  GemmArgs h{};
  h.M = n; h.N = k; h.K = m;
  h.a = p->wt.as<double>(); h.a_is = 1; h.a_ks = n;
  h.b = T; h.b_ks = k; h.b_ns = 1;
  h.c = out; h.c_is = o_rs; h.c_ns = o_cs;
  h.kchunk = m; h.part_stride = 0;
  h.alpha = alpha;
  h.beta = beta;
  h.src = b; h.s_is = b_rs; h.s_ns = b_cs;
  dim3 grid2((unsigned)((n + BM - 1) / BM), (unsigned)((k + BN - 1) / BN), 1);
  dgemm_kernel<<<grid2, GT, 0, st>>>(h);
  KGP_LAUNCH("dgemm_kernel (U T)");
  return KGP_OK;
}

// out = beta B + alpha U (U^T B)
int lowrank_apply_impl(kgp_precond_s* p, double beta, double alpha, int64_t k, const double* b, int64_t b_rs,
                       int64_t b_cs, double* out, int64_t o_rs, int64_t o_cs, cudaStream_t st) {
  int rc = p->tproj.ensure(sizeof(double) * (size_t)p->m * k);
  if (rc) return rc;
  rc = lowrank_project_impl(p, k, b, b_rs, b_cs, p->tproj.as<double>(), st);
  if (rc) return rc;
  return lowrank_expand_impl(p, beta, alpha, k, b, b_rs, b_cs, p->tproj.as<double>(), out, o_rs, o_cs, st);
}

// Woodbury inverse: B / s - W (W^T B) / s^2
int precond_apply_impl(kgp_precond_s* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* out,
                       int64_t o_rs, int64_t o_cs, cudaStream_t st) {
  if (p->kind == KGP_PRECOND_AFN) return afn_apply_impl(p, k, b, b_rs, b_cs, out, o_rs, o_cs, st);
  return lowrank_apply_impl(p, 1.0 / p->s, -1.0 / (p->s * p->s), k, b, b_rs, b_cs, out, o_rs, o_cs, st);
}

}  // namespace kgp
