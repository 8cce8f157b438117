// Symmetric DENSE-mode product for few right-hand sides: out = Khat B, k <= SYM_MAXK.
//
// The reference's DENSE mode (kmat.py:107-123, auto-selected for n <= 20000) multiplies the
// materialised Khat by the RHS every PCG iteration. With one RHS column (the w-solve, and the
// whole narrowed PCG tail) that product is a GEMV over n^2 fp64: 134 MB at configs[0], which
// does not fit the 126 MB L2, so every iteration streams it from HBM (cuBLAS: 25.6 us).
// Khat is exactly symmetric (kappa(x_i, x_j) and kappa(x_j, x_i) are the same rounded
// value), so only its upper triangle is needed: packed into 64 x 64 tiles it is 68 MB, which
// fits the L2 (an explicit persisting access-policy window measured no better). Measured at
// configs[0]: 16.4 us per product against 25.6 us for the cuBLAS GEMV over the full matrix
// (launch lists with warm caches). Each tile (I, J), I <= J, is read ONCE per product
// and gives both its row contribution K_IJ x_J (to y_I) and, off the diagonal, its column
// contribution K_IJ^T x_I (to y_J). Contributions go to a partial buffer Q[I][J] and are
// summed in J order (fixed, so results are run-to-run identical; they differ from a GEMM
// only in summation order).
#include <stdlib.h>

#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

constexpr int ST = 64;  // tile edge

__host__ __device__ inline int64_t sym_tile_index(int64_t I, int64_t J, int64_t nb) {
  return I * nb - I * (I - 1) / 2 + (J - I);  // row-major upper triangle incl. the diagonal
}

// packed[tile(I, J)][a][b] = Khat[I*64 + a][J*64 + b] (zero beyond n)
__global__ void sym_pack_kernel(int64_t n, int64_t nb, const double* __restrict__ dense, double* __restrict__ packed) {
  const int64_t J = blockIdx.x, I = blockIdx.y;
  if (J < I) return;
  double* t = packed + sym_tile_index(I, J, nb) * ST * ST;
  for (int e = threadIdx.x; e < ST * ST; e += blockDim.x) {
    const int64_t r = I * ST + e / ST, c = J * ST + e % ST;
    t[e] = (r < n && c < n) ? dense[r * n + c] : 0.0;
  }
}

// Q[(I nb + J) k + c][a] = (K_IJ x_J)[a];  Q[(J nb + I) k + c][b] = (K_IJ^T x_I)[b] for I < J.
// One CTA per tile (CTAs below the diagonal exit). The tile (32 KB) is loaded with eight
// independent 16-byte loads per thread; row sums: thread (a = t/4, quarter t%4) sums columns
// t%4 + 4j, the quarters combine by shuffles in a fixed order; column sums: thread (b = t%64,
// quarter t/64) sums 16 rows, the quarters combine through shared memory in a fixed order.
// (A persistent variant prefetching the next tile into registers measured slower: 18.8 vs
// 16.4 us per product at n = 4096.)
__global__ void __launch_bounds__(256) sym_tile_kernel(int64_t n, int64_t nb, int k, const double* __restrict__ packed,
                                                       const double* __restrict__ b, int64_t b_cs,
                                                       double* __restrict__ q) {
  const int64_t J = blockIdx.x, I = blockIdx.y;
  if (J < I) return;
  __shared__ double tile[ST][ST + 4];  // row stride 68: the row pass's (a, column) pairs spread over the banks
  __shared__ double xi[SYM_MAXK][ST], xj[SYM_MAXK][ST];
  __shared__ double cpart[4][SYM_MAXK][ST];
  const int tid = threadIdx.x;
  const double2* src = reinterpret_cast<const double2*>(packed + sym_tile_index(I, J, nb) * ST * ST);
  double2 v[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) v[m] = src[tid + 256 * m];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int e = 2 * (tid + 256 * m);
    tile[e / ST][e % ST] = v[m].x;
    tile[e / ST][e % ST + 1] = v[m].y;
  }
  for (int e = tid; e < k * ST; e += 256) {
    const int c = e / ST, a = e % ST;
    const int64_t ri = I * ST + a, rj = J * ST + a;
    xi[c][a] = ri < n ? b[ri + c * b_cs] : 0.0;
    xj[c][a] = rj < n ? b[rj + c * b_cs] : 0.0;
  }
  __syncthreads();
  {  // row sums -> y_I
    const int a = tid >> 2, qt = tid & 3;
    double* dst = q + (I * nb + J) * k * ST;
    for (int c = 0; c < k; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int bb = 0; bb < 16; ++bb) acc = fma(tile[a][qt + 4 * bb], xj[c][qt + 4 * bb], acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);  // (q0 + q1), (q2 + q3): same order in every lane pair
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (qt == 0) dst[c * ST + a] = acc;
    }
  }
  if (I != J) {  // column sums -> y_J
    const int bb = tid & (ST - 1), qt = tid >> 6;
    for (int c = 0; c < k; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 16; ++a) acc = fma(tile[qt * 16 + a][bb], xi[c][qt * 16 + a], acc);
      cpart[qt][c][bb] = acc;
    }
    __syncthreads();
    double* dst = q + (J * nb + I) * k * ST;
    for (int e = tid; e < k * ST; e += 256) {
      const int c = e / ST, b2 = e % ST;
      dst[c * ST + b2] = (cpart[0][c][b2] + cpart[1][c][b2]) + (cpart[2][c][b2] + cpart[3][c][b2]);
    }
  }
}

// out[I*64 + a + c o_cs] = sum_J Q[(I nb + J) k + c][a], J ascending
__global__ void sym_reduce_kernel(int64_t n, int64_t nb, int k, const double* __restrict__ q, double* __restrict__ out,
                                  int64_t o_cs) {
  const int64_t I = blockIdx.x;
  const int c = blockIdx.y, a = threadIdx.x;
  const int64_t r = I * ST + a;
  if (r >= n) return;
  double acc = 0.0;
  int64_t J = 0;
  for (; J + 8 <= nb; J += 8) {  // eight independent loads in flight, added in J order
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = q[((I * nb + J + u) * k + c) * ST + a];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  for (; J < nb; ++J) acc += q[((I * nb + J) * k + c) * ST + a];
  out[r + c * o_cs] = acc;
}

}  // namespace

int64_t sym_packed_elems(int64_t n) {
  const int64_t nb = (n + ST - 1) / ST;
  return nb * (nb + 1) / 2 * ST * ST;
}

int64_t sym_q_elems(int64_t n) {
  const int64_t nb = (n + ST - 1) / ST;
  return nb * nb * SYM_MAXK * ST;
}

int sym_pack(int64_t n, const double* dense, double* packed, cudaStream_t st) {
  const int64_t nb = (n + ST - 1) / ST;
  sym_pack_kernel<<<dim3((unsigned)nb, (unsigned)nb), 256, 0, st>>>(n, nb, dense, packed);
  KGP_LAUNCH("sym_pack_kernel");
  return KGP_OK;
}

int sym_matmul(int64_t n, const double* packed, int k, const double* b, int64_t b_cs, double* out, int64_t o_cs,
               double* q, cudaStream_t st) {
  KGP_REQUIRE(k >= 1 && k <= SYM_MAXK, KGP_ERR_INVALID, "symmetric product takes 1..%d columns", SYM_MAXK);
  const int64_t nb = (n + ST - 1) / ST;
  sym_tile_kernel<<<dim3((unsigned)nb, (unsigned)nb), 256, 0, st>>>(n, nb, k, packed, b, b_cs, q);
  KGP_LAUNCH("sym_tile_kernel");
  sym_reduce_kernel<<<dim3((unsigned)nb, (unsigned)k), ST, 0, st>>>(n, nb, k, q, out, o_cs);
  KGP_LAUNCH("sym_reduce_kernel");
  return KGP_OK;
}

}  // namespace kgp
