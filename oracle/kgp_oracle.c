/*
 * CPU ORACLE (C restatement) — test infrastructure and CPU baseline only.
 *
 * A plain-C, OpenMP restatement of the reference's streamed operator
 * KernelEngine._streamed_matmul (/root/reference/pkg/src/kernelgp/kmat.py:165-189)
 * with the numba panel arithmetic (_panels_numba.py:37-131): per entry a
 * direct-difference r^2, then kappa or d kappa/dl, contracted against the RHS
 * block, scaled by f^2 (or 2f), plus s*B on the diagonal rows.
 *
 * It exists for two reasons: the numpy oracle is too slow for row subsamples at
 * the BASELINE sizes, and bench.py's cpu_baseline / --impl reference legs need
 * the reference algorithm timed on every host core of the GPU box, where the
 * Python reference itself is not present. Only tests/, smoke() and bench.py load
 * it. tests/test_oracle.py pins it against the reference golden vectors.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RB 4   /* rows per register block */

static inline double kappa(int kt, double acc, double l) {
  if (kt == 0) return exp(-acc * (1.0 / (2.0 * l * l)));
  double t = (kt == 1 ? sqrt(3.0) : sqrt(5.0)) / l * sqrt(acc);
  if (kt == 1) return (1.0 + t) * exp(-t);
  return (1.0 + t + (5.0 / (3.0 * l * l)) * acc) * exp(-t);
}

static inline double dkappa(int kt, double acc, double l) {
  if (kt == 0) return acc * (1.0 / (l * l * l)) * exp(-acc * (1.0 / (2.0 * l * l)));
  if (kt == 1) return (3.0 / (l * l * l)) * acc * exp(-(sqrt(3.0) / l) * sqrt(acc));
  double t = (sqrt(5.0) / l) * sqrt(acc);
  return (5.0 / (3.0 * l * l * l)) * acc * (1.0 + t) * exp(-t);
}

int kgpo_version(void) { return 1; }

int kgpo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* out_k[r,:]  = f^2 sum_j kappa(x_{row0+r}, x_j) b[j,:] + s b[row0+r,:]
 * out_dl[r,:] = f^2 sum_j dkappa/dl(x_{row0+r}, x_j) b[j,:]
 * x (n,d) row-major, b (n,k) row-major, outputs (nrows,k) row-major; either may be NULL. */
int kgpo_matmul(int kt, int64_t n, int d, const double* x, double l, double f, double s,
                int64_t row0, int64_t nrows, int64_t k, const double* b,
                double* out_k, double* out_dl, int nthreads) {
  if (kt < 0 || kt > 2 || n < 1 || d < 1 || k < 1 || row0 < 0 || row0 + nrows > n) return 1;
  const double f2 = f * f;
  const int64_t nblk = (nrows + RB - 1) / RB;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
  {
    double* pk = (double*)malloc(sizeof(double) * RB * n);
    double* pg = (double*)malloc(sizeof(double) * RB * n);
    double* acck = (double*)malloc(sizeof(double) * RB * k);
    double* accg = (double*)malloc(sizeof(double) * RB * k);
#pragma omp for schedule(dynamic, 4)
    for (int64_t bi = 0; bi < nblk; ++bi) {
      int64_t r0 = bi * RB;
      int rb = (int)((nrows - r0) < RB ? (nrows - r0) : RB);
      /* panel rows (the numba panel: direct differences, then the transform) */
      for (int r = 0; r < rb; ++r) {
        const double* xi = x + (row0 + r0 + r) * d;
        for (int64_t j = 0; j < n; ++j) {
          const double* xj = x + j * d;
          double acc = 0.0;
          for (int q = 0; q < d; ++q) {
            double diff = xi[q] - xj[q];
            acc += diff * diff;
          }
          if (out_k) pk[r * n + j] = kappa(kt, acc, l);
          if (out_dl) pg[r * n + j] = dkappa(kt, acc, l);
        }
      }
      /* contraction panel . B (the np.dot of kmat.py:185) */
      if (out_k) memset(acck, 0, sizeof(double) * RB * k);
      if (out_dl) memset(accg, 0, sizeof(double) * RB * k);
      for (int64_t j = 0; j < n; ++j) {
        const double* bj = b + j * k;
        for (int r = 0; r < rb; ++r) {
          if (out_k) {
            double v = pk[r * n + j];
            double* a = acck + r * k;
            for (int64_t c = 0; c < k; ++c) a[c] += v * bj[c];
          }
          if (out_dl) {
            double v = pg[r * n + j];
            double* a = accg + r * k;
            for (int64_t c = 0; c < k; ++c) a[c] += v * bj[c];
          }
        }
      }
      for (int r = 0; r < rb; ++r) {
        int64_t gi = row0 + r0 + r;
        for (int64_t c = 0; c < k; ++c) {
          if (out_k) out_k[(r0 + r) * k + c] = f2 * acck[r * k + c] + s * b[gi * k + c];
          if (out_dl) out_dl[(r0 + r) * k + c] = f2 * accg[r * k + c];
        }
      }
    }
    free(pk); free(pg); free(acck); free(accg);
  }
  return 0;
}

/* Materialised rectangular panel (kernels.py:79-94 via the numba panels, _panels_numba.py:37-131,
 * prange over rows): out[i,j] = scale * kappa(x_i, y_j) (which = 0) or scale * dkappa/dl (which = 1),
 * plus `diag` on i == j when add_diag (Khat = f^2 kappa + s I, kmat.py:107-120). Row-major (nx, ny).
 * The reference's DENSE mode (auto for n <= 20000) builds these with every host core; the CPU
 * baseline of the NLML metric does the same here. */
int kgpo_panel(int kt, int which, int64_t nx, int64_t ny, int d, const double* x, const double* y, double l,
               double scale, double diag, int add_diag, double* out, int nthreads) {
  if (kt < 0 || kt > 2 || which < 0 || which > 1 || nx < 0 || ny < 0 || d < 1) return 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nx; ++i) {
    const double* xi = x + i * d;
    double* o = out + i * ny;
    for (int64_t j = 0; j < ny; ++j) {
      const double* yj = y + j * d;
      double acc = 0.0;
      for (int q = 0; q < d; ++q) {
        double diff = xi[q] - yj[q];
        acc += diff * diff;
      }
      o[j] = scale * (which == 0 ? kappa(kt, acc, l) : dkappa(kt, acc, l));
    }
    if (add_diag && i < ny) o[i] += diag;
  }
  return 0;
}
