/*
 * libkgp — C ABI of the B200-native HiGP hot path.
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.
 * Device pointers are CUDA global-memory addresses on the engine's device;
 * `stream` is a cudaStream_t (NULL = legacy default stream). All work is
 * stream-ordered; functions that return host scalars synchronise the stream.
 *
 * Every entry point replaces one reference interface (paths relative to
 * /root/reference/pkg/src/kernelgp/); the citation is next to each declaration.
 *
 * Errors: every function returns KGP_OK (0) or a KGP_ERR_* code; the message
 * is available from kgp_last_error() (thread-local). The Python host maps
 * codes onto the reference exception types (errors.py:4-17).
 */
#ifndef KGP_H_
#define KGP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KGP_ABI_VERSION 1

/* return codes */
#define KGP_OK 0
#define KGP_ERR_INVALID 1   /* -> ValueError            (kernels.py:43-64, kmat.py:62-73) */
#define KGP_ERR_RESOURCE 2  /* -> ResourceLimitError    (kmat.py:111-115)                  */
#define KGP_ERR_BREAKDOWN 3 /* -> BreakdownError        (solver.py:160-164)                */
#define KGP_ERR_NUMERICAL 4 /* -> NumericalError        (solver.py:172-173, 260-263)       */
#define KGP_ERR_CUDA 5      /* -> KernelGpError         (device / launch failure)          */
#define KGP_ERR_STATE 6     /* -> KernelGpError         (use after destroy, double destroy) */

/* kernel ids: KernelType (kernels.py:29-40) */
#define KGP_GAUSSIAN 0
#define KGP_MATERN32 1
#define KGP_MATERN52 2

/* operator arithmetic */
#define KGP_FP64 0  /* fp64 tile, fp64 contraction (parity anchor)                        */
#define KGP_FAST 1  /* fp32 centred tile + 3xTF32 tcgen05 contraction, fp32 TMEM accumulation */
#define KGP_TF32 2  /* fp32 centred tile + 1xTF32 tcgen05 contraction (throughput mode)     */
#define KGP_BF16X3 3 /* fp32 centred tile split into two bf16 terms, contraction A0B0 + A0B1 + A1B0
                        (kind::f16, K=16), fp32 TMEM accumulation (MatMul throughput mode)     */

/* preconditioner kinds (kgp_precond_kind) */
#define KGP_PRECOND_NYSTROM 0
#define KGP_PRECOND_AFN 1

typedef struct kgp_engine_s kgp_engine;
typedef struct kgp_precond_s kgp_precond;

/* ------------------------------------------------------------------ library */
int kgp_version(void);
const char* kgp_last_error(void);
int kgp_device_count(int* count);

/* ------------------------------------------------------------------ engine
 * KernelEngine.__init__ (kmat.py:79-103): Khat = f^2 kappa(X, X; l) + s I with X
 * copied into HBM (the engine never aliases caller data, kmat.py:90).
 * x: (n, d) row-major fp64, host (x_on_device = 0) or device (1). */
int kgp_engine_create(kgp_engine** out, int device, int kernel, int precision, int64_t n, int d,
                      const double* x, int x_on_device, double l, double f, double s, void* stream);
/* Engines are immutable in the reference; hyperparameters are reset here so a
 * training loop (train.py:196-204) reuses the resident X. */
int kgp_engine_set_params(kgp_engine* e, double l, double f, double s, void* stream);
int kgp_engine_set_precision(kgp_engine* e, int precision);
/* Row partition for multi-GPU: this engine produces rows [row0, row0 + nrows) of Khat.B. */
int kgp_engine_set_rows(kgp_engine* e, int64_t row0, int64_t nrows);
int kgp_engine_destroy(kgp_engine* e); /* second destroy of the same handle -> KGP_ERR_STATE */
/* DENSE mode (kmat.py:93-94, 107-123: the reference auto-selects it for n <= 20000):
 * with precision KGP_FP64, single-output products Khat.B (unit-stride columns) use Khat
 * materialised once in HBM (n^2 fp64, rebuilt when (l, f, s) change) and a cuBLAS DGEMM;
 * derivative products stay on the fused kernel. enable = 0 frees the matrix. */
int kgp_engine_set_dense(kgp_engine* e, int enable);
/* Heteroscedastic shift for GP classification (no reference counterpart: SPEC.md:382 lists
 * GPC and heteroscedastic noise as non-goals; the Dirichlet-based GPC of gpc.py needs it):
 * column c of every later Khat product becomes f^2 kappa b_c + (s + dn[map[c]]) o b_c.
 * dn: (classes, n) device fp64, class-major (copied); map: ncols int32 on the HOST (copied);
 * products with more than ncols columns are rejected. classes = 0 removes it. The
 * derivative outputs are unaffected (the diagonal is data, not a hyperparameter). */
int kgp_engine_set_diag(kgp_engine* e, int classes, const double* dn, int64_t ncols, const int32_t* map,
                        void* stream);

/* KernelEngine.matmul / grad_matmul (kmat.py:145-189), fused in one pass:
 *   out_k  = f^2 kappa(X_rows, X) B + s B_rows        (matmul)
 *   out_dl = f^2 dkappa/dl(X_rows, X) B               (grad_matmul Theta.L)
 *   out_df = 2 f kappa(X_rows, X) B                   (grad_matmul Theta.F)
 * Any output may be NULL. B: (n, k) device fp64 with element (i, c) at
 * b[i*b_rs + c*b_cs]; outputs (nrows, k) at o[i*o_rs + c*o_cs]. */
int kgp_engine_matmul(kgp_engine* e, int64_t k, const double* b, int64_t b_rs, int64_t b_cs,
                      double* out_k, double* out_dl, double* out_df, int64_t o_rs, int64_t o_cs,
                      void* stream);

/* The same product on HOST buffers (the reference's numpy-in/numpy-out matmul,
 * kmat.py:145-163): b (n, k) and every requested output (nrows, k) row-major contiguous
 * host fp64 (pinned memory gives asynchronous DMA). The output transfer is pipelined
 * behind the computation in row chunks; returns when the outputs are written. */
int kgp_engine_matmul_host(kgp_engine* e, int64_t k, const double* b, double* out_k, double* out_dl,
                           double* out_df, void* stream);

/* ------------------------------------------------------------------ fused all-gather + operator
 * The multi-GPU row partition (the reference has no multi-GPU path, its
 * product is kmat.py:165-189) without a separate all-gather of the RHS: rank q owns rows
 * [row_start[q], row_start[q+1]) of B (boundaries on multiples of 32) and publishes them,
 * already in the operator's tf32 tile layout, in a buffer every rank maps (CUDA IPC); each
 * rank's operator kernel pulls the owners' tiles (over NVLink) block by block as its column
 * sweep reaches them, so the exchange overlaps the math. Replaces dist.py's NCCL
 * all_gather + K^[I_g, :] P. Per product, epoch e = 1, 2, ...:
 *   kgp_engine_peer_publish: wait until every peer's done >= e - 1 (it finished reading the
 *     previous tiles), write the own tiles, ready = e;
 *   kgp_engine_peer_matmul: the kernel waits for each owner's ready >= e before its first
 *     tile; afterwards done = e.
 * Flags are system-scope release/acquire; waits are bounded (a peer that never arrives
 * traps the kernel -> KGP_ERR_CUDA, never a hang). Buffers: [ready | done | pad to 1 KB]
 * then the tiles; tensor-core precisions only; one launch's RHS block (k). */
int kgp_peer_alloc(int64_t bytes, void** dptr, void* ipc_handle /* 64-byte cudaIpcMemHandle out, or NULL */);
int kgp_peer_open(const void* ipc_handle, void** dptr); /* map a peer's buffer (cudaIpcOpenMemHandle) */
int kgp_peer_close(void* dptr);                         /* unmap an opened peer buffer */
int kgp_peer_free(void* dptr);                          /* free an own kgp_peer_alloc buffer */
int kgp_engine_peer_buffer_bytes(kgp_engine* e, int64_t k, int64_t own_rows, int64_t* bytes);
/* engine rows must already be rank's block (kgp_engine_set_rows); bases[q] = rank q's buffer,
 * sized by kgp_engine_peer_buffer_bytes for RHS blocks of up to k_cap columns */
int kgp_engine_set_peers(kgp_engine* e, int world, int rank, const int64_t* row_start, void* const* bases,
                         int64_t k_cap);
/* b_loc: this rank's rows (nrows x k, strides b_rs / b_cs), valid until the matching peer_matmul */
int kgp_engine_peer_publish(kgp_engine* e, int64_t k, const double* b_loc, int64_t b_rs, int64_t b_cs,
                            uint64_t epoch, void* stream);
int kgp_engine_peer_matmul(kgp_engine* e, int64_t k, uint64_t epoch, double* out_k, double* out_dl, double* out_df,
                           int64_t o_rs, int64_t o_cs, void* stream);

/* Rectangular f^2 kappa(Xs, X) B (no diagonal shift): the cross kernel of predict
 * (gp.py:223-241), never materialised. xs: (m, d) device fp64 row-major. */
int kgp_engine_cross_matmul(kgp_engine* e, int64_t m, const double* xs, int64_t k, const double* b,
                            int64_t b_rs, int64_t b_cs, double* out, int64_t o_rs, int64_t o_cs,
                            void* stream);

/* ------------------------------------------------------------------ panels
 * eval_kernel / eval_kernel_grad_l / pairwise_sq_dist (kernels.py:72-94):
 * out[i*ldo + j] = kappa(x_i, y_j; l) (grad=0), dkappa/dl (grad=1), r^2 (grad=2).
 * x (nx, d), y (ny, d) device row-major fp64. */
int kgp_eval_panel(int kernel, int grad, int64_t nx, int64_t ny, int d, const double* x, const double* y,
                   double l, double* out, int64_t ldo, void* stream);

/* fps_select (precond.py:39-59): greedy farthest-point sampling from seed_index,
 * ties to the lowest index. x (n, d) device; idx_out: m int64 on the device. */
int kgp_fps(int64_t n, int d, const double* x, int64_t m, int64_t seed_index, int64_t* idx_out,
            void* stream);

/* ------------------------------------------------------------------ preconditioner
 * NystromPreconditioner.apply_inverse (precond.py:74-83) in factored Woodbury form
 *   M^-1 B = B / s - W (W^T B) / s^2,   W = V L_C^-T,  C = I/f^2 + V^T V / s = L_C L_C^T
 * wt: W^T as (m, n) row-major device fp64 (copied). */
int kgp_precond_create(kgp_precond** out, int64_t n, int64_t m, const double* wt, double s, void* stream);
int kgp_precond_destroy(kgp_precond* p);
/* B and out: (n, k) strided device fp64 as in kgp_engine_matmul. */
int kgp_precond_apply_inverse(kgp_precond* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs,
                              double* out, int64_t o_rs, int64_t o_cs, void* stream);

/* NystromPreconditioner.apply (precond.py:85-92) and any symmetric low-rank update:
 * out = beta B + alpha U (U^T B), with U^T the handle's (m, n) factor. A handle
 * created from V^T with beta = s, alpha = f^2 applies M itself. */
int kgp_lowrank_apply(kgp_precond* p, double beta, double alpha, int64_t k, const double* b, int64_t b_rs,
                      int64_t b_cs, double* out, int64_t o_rs, int64_t o_cs, void* stream);

/* The two halves of kgp_lowrank_apply, for a row-partitioned factor (multi-GPU):
 * project: t_out = U^T B, (m, k) row-major device (the caller all-reduces it across ranks);
 * expand:  out = beta B + alpha U t. The handle then holds only this rank's rows of U. */
int kgp_lowrank_project(kgp_precond* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* t_out,
                        void* stream);
int kgp_lowrank_expand(kgp_precond* p, double beta, double alpha, int64_t k, const double* b, int64_t b_rs,
                       int64_t b_cs, const double* t, double* out, int64_t o_rs, int64_t o_cs, void* stream);

/* ------------------------------------------------------------------ AFN preconditioner
 * The north star's "AFN preconditioner applied on device (landmark Cholesky solve plus
 * sparse FSAI factor matvec)". The reference substitutes Nystrom for AFN
 * ("the module interface (build/apply_inverse) is exactly what an
 * AFN drop-in would implement"), so these entries extend precond.py's build/apply_inverse
 * pair; an AFN handle is accepted wherever a kgp_precond is (kgp_precond_apply_inverse,
 * kgp_pcg, kgp_nlml_grad). Ordering: m landmarks first, then the n2 = n - m others.
 *
 * kgp_knn_prev: for each point i of x (n, d) device fp64, the npt (<= 64) nearest points
 *   j < i by squared distance, ties to the lower j, nearest first; idx_out (n, npt) int64
 *   device, -1 padded (the FSAI sparsity pattern).
 * kgp_afn_fsai: row i of the FSAI factor G of S = Khat22 - W W^T on the pattern
 *   {nbr[i, :], i}: gval/gcol (npt + 1, n2) slot-major (entry t of row i at t*n2 + i),
 *   the diagonal last, -1/0 padded. x2 (n2, d) the non-landmark points, w (n2, m)
 *   row-major. dshift (n2) adds a per-point diagonal to S (heteroscedastic noise, gpc.py;
 *   NULL: none). A non-SPD pattern block -> KGP_ERR_BREAKDOWN.
 * kgp_afn_create: handle from device factors (all copied): perm (n) permuted position ->
 *   original row, linv (m, m) row-major L11^-1, l11 (m, m) L11 itself (NULL: no sampling),
 *   w (n2, m), the ELL factor from
 *   kgp_afn_fsai, and G^T as CSR (gtptr n2 + 1, gtrow/gtval nnz; rows ascending). */
int kgp_knn_prev(int64_t n, int d, const double* x, int npt, int64_t* idx_out, void* stream);
int kgp_afn_fsai(int kernel, int64_t n2, int d, const double* x2, double l, double f, double s,
                 const double* dshift, int64_t m, const double* w, int npt, const int64_t* nbr, double* gval,
                 int32_t* gcol, void* stream);
int kgp_afn_create(kgp_precond** out, int64_t n, int64_t m, const int64_t* perm, const double* linv,
                   const double* l11, const double* w, int npt1, const double* gval, const int32_t* gcol,
                   int64_t nnz, const int32_t* gtptr, const int32_t* gtrow, const double* gtval, double s,
                   void* stream);
/* z ~ N(0, M) from standard normals for the preconditioned-probe estimator (kgp_nlml_grad_pp):
 * with w = [w1 (m rows); w2 (n2 rows)] in the landmark-first order, z = L F w with
 * F = diag(L11, G^-1): z1 = L11 w1, z2 = W w1 + G^-1 w2 (forward substitution scheduled by
 * dependency level), scattered back to the original row order. w (n, k) strided device;
 * z (k, n) device, draw c contiguous. Needs the handle created with l11. */
int kgp_afn_sample(kgp_precond* p, int64_t k, const double* w, int64_t w_rs, int64_t w_cs, double* z,
                   void* stream);
int kgp_precond_kind(kgp_precond* p, int* kind);

/* ------------------------------------------------------------------ local predictive variance
 * Large-m prediction variance (an extension; the reference computes the exact variance,
 * gp.py:240-243, one solve per test point): var(x*) ~= f^2 - c^T (Khat_NN)^-1 c over the
 * npt (<= 64) nearest training points N of x* (local kriging). kgp_knn_cross: idx_out
 * (nq, npt) int64 nearest training rows of each query (ties to the lower index);
 * kgp_local_variance: var (nq) from those lists. xq (nq, d), x (nx, d) device fp64. */
int kgp_knn_cross(int64_t nq, const double* xq, int64_t nx, const double* x, int d, int npt, int64_t* idx_out,
                  void* stream);
int kgp_local_variance(int kernel, int64_t nq, int d, const double* xq, const double* x, double l, double f,
                       double s, int npt, const int64_t* nbr, double* var, void* stream);

/* ------------------------------------------------------------------ solvers
 * pcg_solve (solver.py:122-192): batched PCG, per-column alpha/beta capture,
 * converged columns freeze in place. y and x_out: (k, n) device (column c
 * contiguous, the reference's transposed state, solver.py:143-146).
 * alphas/betas: (k, max_iter) device; iters, converged: k int32 device; rel: k fp64.
 * precond may be NULL (unpreconditioned). Breakdown -> KGP_ERR_BREAKDOWN. */
int kgp_pcg(kgp_engine* e, kgp_precond* p, int64_t k, const double* y, double tol, int32_t max_iter,
            double* x_out, double* alphas, double* betas, int32_t* iters, double* rel, int32_t* converged,
            void* stream);

/* kgp_pcg over two column groups sharing one operator application per iteration:
 * columns [0, kpc) preconditioned (tol1, at most it1 iterations), [kpc, k) unpreconditioned
 * (tol2, it2). pcs: 0, 1 (shared by the group) or kpc handles (one per column, e.g. one
 * per GPC class). alphas/betas: (k, max(it1, it2)). The engine's kgp_engine_set_diag
 * state, if any, applies (it must map k columns). */
int kgp_pcg_grouped(kgp_engine* e, kgp_precond* const* pcs, int npcs, int64_t k, int64_t kpc, const double* y,
                    double tol1, int32_t it1, double tol2, int32_t it2, double* x_out, double* alphas,
                    double* betas, int32_t* iters, double* rel, int32_t* converged, void* stream);

/* slq_logdet (solver.py:238-265): per-probe e1^T log(T) e1 from the CG
 * coefficients on the device; returns the probe mean of |z|^2 e1^T log(T) e1 in
 * *logdet (host). norms_sq: k fp64 device. Non-positive Ritz value -> KGP_ERR_NUMERICAL. */
int kgp_slq_logdet(int64_t k, int32_t max_iter, const double* alphas, const double* betas,
                   const int32_t* iters, const double* norms_sq, double* logdet, void* stream);

/* nlml_grad_iterative (gp.py:133-179) end to end on the device:
 * out[0..3] = loss, grad_l, grad_f, grad_s (host); out_converged (host).
 * y: n device; probes: (k_z, n) device (probe c contiguous). probe_max_iter caps the
 * probe CG / Lanczos length separately (<= 0: max_iter, the reference's single knob);
 * with tol = probe_tol = 0 this is BASELINE configs[0]'s fixed recipe (PCG 50, SLQ 20). */
int kgp_nlml_grad(kgp_engine* e, kgp_precond* p, const double* y, int64_t k_z, const double* probes,
                  double tol, int32_t max_iter, double probe_tol, int32_t probe_max_iter, double* out,
                  int32_t* out_converged, void* stream);

/* ------------------------------------------------------------------ instrumentation (bench.py; no reference counterpart)
 * kgp_launch_count: kernels this library has launched in this process (graph replays
 * counted per kernel node). kgp_engine_set_timing(e, 1) brackets every launch of the
 * tensor-core operator kernel with CUDA events on its stream; kgp_engine_kernel_time
 * synchronises, returns the summed kernel time (ms) and the bracketed launch count
 * since the previous read, and resets them. */
int64_t kgp_launch_count(void);
int kgp_engine_set_timing(kgp_engine* e, int enable);
int kgp_engine_kernel_time(kgp_engine* e, double* ms, int64_t* launches);

/* nlml_grad_iterative with PRECONDITIONED probes (an extension; the reference's probes are
 * unpreconditioned, gp.py:154-160): the caller draws probes z ~ N(0, M) for the handle's
 * M and passes logdet_m = log|M|. Probe solves are preconditioned by M, SLQ estimates
 * log|M^-1/2 Khat M^-1/2| (weights z^T M^-1 z) and the trace terms use
 * E[(M^-1 z)^T dK Khat^-1 z] = tr(Khat^-1 dK): unbiased for the same loss and gradient,
 * with probe CG counts of the preconditioned system. p is M (probes); p_w, if not NULL,
 * preconditions the w-solve instead (e.g. AFN for w, Nystrom for the probes, whose N(0, M)
 * draws are cheap). Other arguments as kgp_nlml_grad. */
int kgp_nlml_grad_pp(kgp_engine* e, kgp_precond* p_w, kgp_precond* p, const double* y, int64_t k_z,
                     const double* probes, double logdet_m, double tol, int32_t max_iter, double probe_tol,
                     int32_t probe_max_iter, double* out, int32_t* out_converged, void* stream);

/* Dirichlet GP classification (gpc.py; no reference counterpart): `classes`
 * GP regressions sharing (l, f, s), class c with Khat + diag(dn_c) and target y_c, solved
 * together (one operator application per iteration serves every class's target and
 * probe columns). dn, y: (classes, n) device, class-major; probes (classes * k_z, n)
 * device, class c's probes at rows [c*k_z, (c+1)*k_z). pcs: 0, 1 (shared) or `classes`
 * preconditioner handles (AFN/Nystrom built for class c's diagonal). out[0..3] = summed
 * loss, grad_l, grad_f, grad_s (host). Replaces any kgp_engine_set_diag state; on return
 * the engine has none. */
int kgp_gpc_nlml_grad(kgp_engine* e, int classes, kgp_precond* const* pcs, int npcs, const double* dn,
                      const double* y, int64_t k_z, const double* probes, double tol, int32_t max_iter,
                      double probe_tol, int32_t probe_max_iter, double* out, int32_t* out_converged,
                      void* stream);

/* kgp_gpc_nlml_grad with preconditioned probes: class c's probes (rows [c*k_z, (c+1)*k_z)
 * of `probes`) are draws from N(0, M_c) for pcs[c] (one handle per class, e.g.
 * kgp_afn_sample of an AFN built for Khat + diag(dn_c)), logdet_m = sum_c log|M_c|. */
int kgp_gpc_nlml_grad_pp(kgp_engine* e, int classes, kgp_precond* const* pcs, const double* dn, const double* y,
                         int64_t k_z, const double* probes, double logdet_m, double tol, int32_t max_iter,
                         double probe_tol, int32_t probe_max_iter, double* out, int32_t* out_converged,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KGP_H_ */
