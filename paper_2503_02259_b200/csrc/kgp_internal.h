// Internal (non-ABI) declarations shared by the libkgp translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/kgp.h"

namespace kgp {

constexpr int KGP_MAX_PEERS = 8;     // ranks of a fused all-gather operator (one node)
constexpr int PEER_HDR = 1024;       // peer buffer: [ready u64 | done u64 | pad] then the tiles

// ------------------------------------------------------------------ fast (tcgen05) operator
struct TcParams {
  const float* xrow;      // (nrows, dpad+1): [q_i, u_i0 .. u_i(dpad-1)]
  const float* xcol;      // nblk x (dpad+1) x 32: per 32-column block [q_j | v_j0 | ...]
  const uint8_t* bsplit;  // nblk x TPO x kp x 128 B: RHS tiles, tf32 hi (/lo), swizzled K-major
  int64_t nrows;
  int nblk;
  int nper;               // column blocks per CTA along grid.y (column split)
  int tbeg;               // first column block of this launch (grid.y sweeps [tbeg, nblk)); 0 normally
  int slot0;              // partial-sum slot of grid.y = 0 (column-chunked launches share one part buffer)
  int noreduce;           // 1: leave the partials for a later launch's tc_reduce (more column chunks follow)
  float* part;            // split partial sums (nsplit x nrows x nout*kp); nullptr: no split
  int kp;                 // padded RHS count (multiple of 16, <= 128)
  int k;                  // true RHS count in this launch
  int nsa;                // TMEM A-stage ring depth
  int nsb;                // shared-memory ring depth (set at launch)
  int nab;                // TMEM accumulator buffers: 2 (drain overlaps the MMA) or 1 (wider kp)
  int lb;                 // LB layout (tc_lb_mode): A lo parts in bf16, bf16 lo*hi correction, 3 A stages
  int flush;              // blocks per TMEM accumulation segment before promotion to fp32 smem
  unsigned long long* trace;  // diagnostic (env KGP_TC_TRACE=path): clock64 per pipeline event of CTA (0,0)
  int debug;              // diagnostic bit flags (env KGP_TC_DEBUG): 1 no contraction MMA, 2 no distance MMA, 4 no transform
  double f2, s, two_f, scale_dl;
  const double* b;        // original fp64 RHS (for + s B)
  int64_t b_rs, b_cs;
  int64_t diag_row0;      // global row of local row 0 for the shift; < 0: no shift
  double *out_k, *out_dl, *out_df;
  int64_t o_rs, o_cs;
  cudaEvent_t ev_start, ev_stop;  // host side: optional timing bracket around the main kernel
  // fused all-gather (kgp_engine_peer_matmul): npeer > 0 -> the RHS tiles of column block g
  // come from the owner rank q's published buffer ptile[q] (block g - pblk0[q]), read after
  // that rank's ready flag reaches `epoch`
  const int32_t* gate;    // non-NULL: skip the launch when *gate == 0 (PCG: no active column left)
  int npeer;
  int pblk0[KGP_MAX_PEERS + 1];
  const uint8_t* ptile[KGP_MAX_PEERS];
  const unsigned long long* pready[KGP_MAX_PEERS];
  unsigned long long epoch;
  unsigned long long ptimeout_ns;  // bounded peer-flag wait (KGP_PEER_TIMEOUT_S, default 600 s)
};
int tc_pad_dim(int d);
int tc_max_kp(int dpad, int nout, int split, int nab);
int tc_col_split(int64_t nrows, int nblk, int maxsplit);
int tc_nsa(int dpad, int nout, int split, int kp);
int tc_lb_mode(int dpad, int nout, int split, int kp);
int tc_lb_nab(int mode, int kp);
int tc_rhs_block_bytes(int split, bool lb, int kp);
int tc_split_of(int precision);
int tc_col_block_bytes(int dpad);
bool tc_direct(int dpad);
int tc_dist_mode(int dpad);  // 0 direct differences, 1 tensor-core expansion, 2 FP32 expansion
int launch_kmm_tc(int kt, int dpad, int nout, int split, const TcParams& p, cudaStream_t st);

// ------------------------------------------------------------------ fp64 operator
struct F64Params {
  const double* xr;       // (nrows, d) row points
  const double* xc;       // (ncols, d) column points
  int64_t nrows, ncols;
  int d, k;
  double l, f2, s, two_f, f2_dl;
  const double* b;
  int64_t b_rs, b_cs;
  int64_t diag_row0;
  double *out_k, *out_dl, *out_df;
  int64_t o_rs, o_cs;
  int64_t jchunk;          // columns per grid.z split (set by launch_kmm_f64)
  const int32_t* gate;     // non-NULL: skip the launch when *gate == 0 (PCG: no active column left)
  double* part;            // split partials (set by launch_kmm_f64)
  int64_t part_stride;
};
struct DevBuf;
int launch_kmm_f64(int kt, const F64Params& p, DevBuf& ws, cudaStream_t st);

// ------------------------------------------------------------------ preprocessing (prep.cu)
int prep_rows(int kt, int precision_split, int d, int dpad, int64_t nrows, const double* x, const double* mean,
              double l, float* out, cudaStream_t st);
int prep_cols(int kt, int d, int dpad, int64_t n, const double* x, const double* mean, double l, float* out,
              cudaStream_t st);
int prep_rhs(int split, int lb, int64_t n, int64_t k, int64_t c0, int kp, const double* b, int64_t b_rs, int64_t b_cs,
             uint8_t* out, cudaStream_t st, int blk0 = 0, int blk1 = -1);
int col_mean(int64_t n, int d, const double* x, double* mean, cudaStream_t st);

// ------------------------------------------------------------------ symmetric DENSE product (symv.cu)
constexpr int SYM_MAXK = 4;  // right-hand sides handled by the packed-triangle product
int64_t sym_packed_elems(int64_t n);
int64_t sym_q_elems(int64_t n);
int sym_pack(int64_t n, const double* dense, double* packed, cudaStream_t st);
int sym_matmul(int64_t n, const double* packed, int k, const double* b, int64_t b_cs, double* out, int64_t o_cs,
               double* q, cudaStream_t st);

// ------------------------------------------------------------------ device buffer helper
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes);
  void release();
  ~DevBuf() { release(); }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

// Incremented whenever any device buffer is (re)allocated or freed, or an engine's
// parameters change: captured CUDA graphs record the epoch they were built at and are
// re-captured when it moved (their kernel arguments hold raw pointers and parameters).
void count_launches(int64_t n);
uint64_t graph_epoch();
void bump_graph_epoch();

struct PcgGraph {
  cudaGraphExec_t exec = nullptr;
  int64_t k = 0;
  std::vector<const void*> pcs;
  const void* tail = nullptr;
  int64_t probe_kz = 0;
  int64_t kpc = 0, kz = 0;
  double tol1 = 0.0, tol2 = 0.0;
  int it1 = 0, it2 = 0;
  uint64_t epoch = 0;
  int64_t kernels = 0;  // kernel nodes per replay (launch accounting)
};
constexpr int PCG_LOOKAHEAD = 6;

}  // namespace kgp

// ------------------------------------------------------------------ opaque handles
struct kgp_engine_s {
  uint64_t magic;
  int device, kt, precision, d, dpad;
  int64_t n, row0, nrows;
  double l, f, s;
  kgp::DevBuf x64;   // (n, d) fp64 points
  kgp::DevBuf mean;  // d
  kgp::DevBuf xrow;  // fast path row data for the engine's own rows
  kgp::DevBuf xcol;  // fast path column tiles
  kgp::DevBuf xrow_cross;  // scratch for cross (prediction) rows
  kgp::DevBuf bsplit;      // per-call RHS split
  kgp::DevBuf f64part;     // fp64 operator column-split partials
  kgp::DevBuf tcpart;      // fast operator column-split partials
  // fused all-gather (kgp_engine_set_peers): rank `prank` of `pworld`, rows prow[q]..prow[q+1]
  // of B owned by rank q, whose buffer (flags + tiles) is mapped at pbase[q]
  int pworld = 0, prank = 0, pprec = 0;
  unsigned long long ptimeout_ns = 0;
  int64_t prow[kgp::KGP_MAX_PEERS + 1] = {};
  uint8_t* pbase[kgp::KGP_MAX_PEERS] = {};
  const double* pb = nullptr;  // own rows of B from the last publish (the + s B term)
  int64_t pb_rs = 0, pb_cs = 0, pk = 0, pkcap = 0;
  // set by the PCG driver while it captures its iteration graph: the active-column count the
  // operator launches check first, so iterations replayed past convergence skip the product
  const int32_t* gate = nullptr;
  bool prepared;
  // PCG workspace (grown on demand) and a pinned status word for the per-iteration readback
  kgp::DevBuf ws;
  kgp::DevBuf ws_nlml;     // NLML+gradient workspace
  int32_t* hstatus;
  // captured PCG iteration graphs and their polling state (pcg.cu)
  kgp::PcgGraph gcache[4];
  int gnext = 0;
  int32_t* hist_host = nullptr;  // mapped pinned (active, error) per iteration
  int32_t* hist_dev = nullptr;
  int hist_cap = 0;
  cudaEvent_t events[kgp::PCG_LOOKAHEAD] = {};
  cudaStream_t cstream = nullptr;  // private stream used only for graph capture (the caller's may be legacy)
  // host-buffer products (kgp_engine_matmul_host): device staging, copy stream, chunk events
  kgp::DevBuf hostbuf;
  cudaStream_t xstream = nullptr;
  cudaEvent_t xev[8] = {};
  cudaEvent_t zev[9] = {};   // host entry: H2D chunks of the RHS (8) + "stream ready" (1)
  // optional heteroscedastic diagonal (kgp_engine_set_diag): Khat column c gets + diag(dn[:, dmap[c]])
  int dn_classes = 0;
  int64_t dn_ncols = 0;
  kgp::DevBuf dn;    // (classes, n): class-major
  kgp::DevBuf dmap;  // dn_ncols int32: RHS column -> class
  // DENSE mode (kgp_engine_set_dense): Khat materialised once, products by cuBLAS DGEMM
  bool dense_on = false, dense_valid = false;
  kgp::DevBuf dense;        // (n, n) fp64 Khat = f^2 kappa + s I
  kgp::DevBuf dpack;        // upper triangle of Khat in 64 x 64 tiles (symv.cu), L2-resident
  kgp::DevBuf dq;           // partial sums of the packed product
  void* cublas = nullptr;   // cublasHandle_t
  // optional main-kernel timing (kgp_engine_set_timing)
  bool timing = false;
  std::vector<cudaEvent_t> tev;  // start/stop pairs
  size_t tev_used = 0;
};

struct kgp_precond_s {
  uint64_t magic;
  int kind;          // KGP_PRECOND_NYSTROM or KGP_PRECOND_AFN
  int64_t n, m;      // m: rank (Nystrom) / landmark count (AFN)
  double s;
  kgp::DevBuf wt;    // Nystrom: (m, n) row-major
  kgp::DevBuf tmp;   // split-K partials
  kgp::DevBuf tproj; // (m, k) projection U^T B
  kgp::DevBuf tmp2;  // expansion partials (kept apart from tmp: the projection result may live there)
  // AFN (afn.cu): landmarks first, then the rest (n2 = n - m points)
  int64_t n2 = 0, nnz = 0;
  int npt1 = 0;       // FSAI row width (neighbours + the diagonal)
  kgp::DevBuf perm;   // n int64: permuted position -> original row
  kgp::DevBuf linv;   // (m, m) row-major L11^-1
  kgp::DevBuf w;      // (n2, m) row-major K21 L11^-T
  kgp::DevBuf gval;   // (npt1, n2) FSAI values, slot-major
  kgp::DevBuf gcol;   // (npt1, n2) int32 columns (-1 padding)
  kgp::DevBuf gtptr;  // n2 + 1 int32: CSR of G^T
  kgp::DevBuf gtrow;  // nnz int32
  kgp::DevBuf gtval;  // nnz
  kgp::DevBuf work;   // apply workspace
  kgp::DevBuf l11;    // (m, m) row-major landmark Cholesky factor (sampling; optional)
  kgp::DevBuf swork;  // sampling workspace
  kgp::DevBuf lvl_rows;             // FSAI rows grouped by dependency level
  std::vector<int64_t> lvl_ptr;     // level offsets into lvl_rows (host)
};

namespace kgp {
constexpr uint64_t ENGINE_MAGIC = 0x6b67702d656e6731ull;
constexpr uint64_t PRECOND_MAGIC = 0x6b67702d70726531ull;
constexpr uint64_t DEAD_MAGIC = 0xdeaddeaddeaddeadull;

int engine_prepare(kgp_engine_s* e, cudaStream_t st);
int engine_matmul_impl(kgp_engine_s* e, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* out_k,
                       double* out_dl, double* out_df, int64_t o_rs, int64_t o_cs, cudaStream_t st);
int lowrank_project_impl(kgp_precond_s* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* T,
                         cudaStream_t st);
int lowrank_expand_impl(kgp_precond_s* p, double beta, double alpha, int64_t k, const double* b, int64_t b_rs,
                        int64_t b_cs, const double* T, double* out, int64_t o_rs, int64_t o_cs, cudaStream_t st);
int lowrank_apply_impl(kgp_precond_s* p, double beta, double alpha, int64_t k, const double* b, int64_t b_rs,
                       int64_t b_cs, double* out, int64_t o_rs, int64_t o_cs, cudaStream_t st);
int precond_apply_impl(kgp_precond_s* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* out,
                       int64_t o_rs, int64_t o_cs, cudaStream_t st);
int afn_apply_impl(kgp_precond_s* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* out,
                   int64_t o_rs, int64_t o_cs, cudaStream_t st);
// C (M x N) = alpha A B + beta SRC with arbitrary strides (fp64, deterministic split-K)
int gemm_f64(int64_t M, int64_t N, int64_t K, const double* a, int64_t a_is, int64_t a_ks, const double* b,
             int64_t b_ks, int64_t b_ns, double* c, int64_t c_is, int64_t c_ns, double alpha, double beta,
             const double* src, int64_t s_is, int64_t s_ns, DevBuf& tmp, cudaStream_t st);

// the AFN application's W products for point-major blocks (wgemm.cu, DMMA):
//   wy:  C = alpha W Y + beta S      (W n2 x m row-major, C n2 x k)
//   wtu: Z = alpha W^T U + beta SRC  (Z m x k), fixed-order row-split partials in tmp
bool wgemm_supported(int64_t m, int64_t k, const double* w, int64_t ldw);
int wy_product(int64_t n2, int64_t m, int64_t k, const double* w, int64_t ldw, const double* y, int64_t y_rs,
               int64_t y_cs, double* c, int64_t c_rs, int64_t c_cs, double alpha, double beta, const double* s,
               int64_t s_rs, int64_t s_cs, cudaStream_t st);
int wtu_product(int64_t n2, int64_t m, int64_t k, const double* w, int64_t ldw, const double* u, int64_t u_rs,
                int64_t u_cs, double* z, int64_t z_rs, int64_t z_cs, double alpha, double beta, const double* src,
                int64_t s_rs, int64_t s_cs, DevBuf& tmp, cudaStream_t st);

// column-wise reductions / updates used by the PCG driver (pcg.cu)
int pcg_solve_impl(kgp_engine_s* e, kgp_precond_s* pc, int64_t k, const double* y, double tol, int max_iter,
                   double* x_out, double* alphas, double* betas, int32_t* iters, double* rel, int32_t* conv,
                   cudaStream_t st);
// PCG over two column groups sharing one operator application per iteration:
// [0, kpc) preconditioned (tol1, cap it1), [kpc, k) unpreconditioned (tol2, cap it2);
// alpha/beta arrays have per-column stride max(it1, it2).
struct PcSet {
  kgp_precond_s* const* h;
  int count;  // 0: none; 1: one handle for every preconditioned column; kpc: one per column
  kgp_precond_s* tail = nullptr;  // precond_all: handle of columns [kpc, k) (default h[0])
  int64_t probe_kz = 0;           // precond_all with one handle per class: probe blocks of this width
};
int pcg_grouped_impl(kgp_engine_s* e, const PcSet& pcs, int64_t k, int64_t kpc, const double* y, double tol1,
                     int it1, double tol2, int it2, double* x_out, double* alphas, double* betas, int32_t* iters,
                     double* rel, int32_t* conv, cudaStream_t st, bool precond_all = false);
int slq_impl(int64_t k, int max_iter, const double* alphas, const double* betas, const int32_t* iters,
             const double* norms_sq, double* logdet, cudaStream_t st);
int col_dots(int64_t k, int64_t n, const double* a, const double* b, double* out, double* partial, cudaStream_t st);
}  // namespace kgp
