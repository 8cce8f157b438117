// C ABI: library, engine and preconditioner handles (include/kgp.h).
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <mutex>
#include <set>
#include <vector>

#include <cublas_v2.h>

#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

static thread_local char g_err_msg[1024] = "";

void set_error(int code, const char* fmt, ...) {
  (void)code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err_msg, sizeof(g_err_msg), fmt, ap);
  va_end(ap);
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return KGP_OK;
  set_error(KGP_ERR_CUDA, "CUDA error in %s: %s", what, cudaGetErrorString(e));
  return KGP_ERR_CUDA;
}

static std::atomic<int64_t> g_launches{0};
void count_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static std::atomic<uint64_t> g_graph_epoch{1};
uint64_t graph_epoch() { return g_graph_epoch.load(); }
void bump_graph_epoch() { g_graph_epoch.fetch_add(1); }

int DevBuf::ensure(size_t bytes) {
  if (bytes <= cap && p) return KGP_OK;
  release();
  bump_graph_epoch();
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    p = nullptr;
    cap = 0;
    (void)cudaGetLastError();
    set_error(KGP_ERR_RESOURCE, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    return KGP_ERR_RESOURCE;
  }
  cap = bytes;
  return KGP_OK;
}

void DevBuf::release() {
  if (p) {
    cudaFree(p);
    bump_graph_epoch();
  }
  p = nullptr;
  cap = 0;
}

double tc_kernel_gamma(int kt, double l);

static void engine_free_host_state(kgp_engine_s* e) {
  if (e->hstatus) cudaFreeHost(e->hstatus);
  if (e->hist_host) cudaFreeHost(e->hist_host);
  for (auto& g : e->gcache)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& ev : e->events)
    if (ev) cudaEventDestroy(ev);
  if (e->cstream) cudaStreamDestroy(e->cstream);
  if (e->xstream) cudaStreamDestroy(e->xstream);
  if (e->cublas) cublasDestroy((cublasHandle_t)e->cublas);
  for (auto ev : e->xev)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : e->zev)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : e->tev) cudaEventDestroy(ev);
}

#ifndef KGP_HOST_CHUNKS_DEFAULT
#define KGP_HOST_CHUNKS_DEFAULT 3
#endif
#ifndef KGP_HOST_RRATIO_DEFAULT
#define KGP_HOST_RRATIO_DEFAULT 50
#endif
static int tc_env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}

// blocks (x32 columns) accumulated in TMEM before promotion: 8 with two accumulator buffers
// (the drain overlaps the MMA), 16 with one (each promotion stalls the MMA: k = 64 two
// outputs 4.93 -> 4.62 ms; error 2.7e-6 -> 3.9e-6, tools/flush_sweep.py). 16 with two buffers
// is 0.6 % faster at cfg2 but its operator error (4.3e-6) put the fast-mode configs[0] NLML
// grad_f at 2.7e-3, over the 1e-3 bar (8: 4.2e-4; tools/nlml_precision.py), so 8 stays.
// Env KGP_TC_FLUSH overrides both.
static int tc_flush_blocks(int nab) {
  static int v = [] {
    const char* s = getenv("KGP_TC_FLUSH");
    int f = s ? atoi(s) : 0;
    return f < 0 ? 0 : f;
  }();
  return v > 0 ? v : (nab == 1 ? 16 : 8);
}

static std::mutex g_handles_mu;
static std::set<const void*> g_handles;

static bool handle_live(const void* h) {
  std::lock_guard<std::mutex> g(g_handles_mu);
  return g_handles.count(h) != 0;
}

int engine_prepare(kgp_engine_s* e, cudaStream_t st) {
  if (e->prepared || e->precision == KGP_FP64) return KGP_OK;
  const int dp = e->dpad;
  int nblk = (int)((e->n + 31) / 32);
  int rc = e->xcol.ensure((size_t)nblk * tc_col_block_bytes(dp));
  if (rc) return rc;
  rc = e->xrow.ensure(sizeof(float) * (size_t)(e->nrows + 1) * (dp + 1));
  if (rc) return rc;
  rc = prep_cols(e->kt, e->d, dp, e->n, e->x64.as<double>(), e->mean.as<double>(), e->l, e->xcol.as<float>(), st);
  if (rc) return rc;
  rc = prep_rows(e->kt, 0, e->d, dp, e->nrows, e->x64.as<double>() + e->row0 * e->d, e->mean.as<double>(), e->l,
                 e->xrow.as<float>(), st);
  if (rc) return rc;
  e->prepared = true;
  return KGP_OK;
}

static double scale_dl_fast(int kt, double l, double f) {
  double f2 = f * f;
  if (kt == GAUSS) return f2 / (tc_kernel_gamma(kt, l) * l * l * l);
  if (kt == MAT32) return f2 / l;
  return f2 / (3.0 * l);
}

// tcgen05 contraction scheme of a tensor-core precision: 3 = 3xTF32, 1 = 1xTF32, 2 = bf16x3
int tc_split_of(int precision) { return precision == KGP_FAST ? 3 : precision == KGP_BF16X3 ? 2 : 1; }

// Shared by the square operator (xrow = engine rows, shift on) and the cross operator.
// skip_prep: the RHS split of exactly this B is already in e->bsplit (row-chunked host
// products prepare it once for all chunks; valid when k fits one launch)
// Column chunk of a pipelined product (kgp_engine_matmul_host): this launch sweeps column blocks
// [blk0, blk1) only, writing fp32 partials into slots [slot0, slot0 + used) of a buffer sized for
// `slots_total`; the last chunk (reduce) sums every slot in order.
struct ColChunk {
  int blk0, blk1, slot0, slots_total;
  bool reduce;
  int used;  // out: slots this chunk wrote
};
static int tc_col_chunk_splits(int64_t nrows, int nblocks) {
  return tc_col_split(nrows, nblocks, tc_env_int("KGP_TC_MAXSPLIT", 16));
}

static int tc_matmul(kgp_engine_s* e, const float* xrow, int64_t nrows, int64_t diag_row0, int64_t k, const double* b,
                     int64_t b_rs, int64_t b_cs, double* out_k, double* out_dl, double* out_df, int64_t o_rs,
                     int64_t o_cs, cudaStream_t st, bool skip_prep = false, uint64_t peer_epoch = 0,
                     ColChunk* cc = nullptr) {
  // peer_epoch > 0: fused all-gather -- the RHS tiles come from the ranks' published buffers
  // (kgp_engine_peer_publish), b is this rank's own rows (diag_row0 = 0 indexes them)
  const int split = tc_split_of(e->precision);
  const int nout = out_dl ? 2 : 1;
  const int nblk = (int)((e->n + 31) / 32);
  // two accumulator buffers when the RHS block fits, else one (the drain then briefly
  // stalls the MMA every `flush` blocks, still far cheaper than a second pass)
  const int kmax2 = tc_max_kp(e->dpad, nout, split, 2);
  const int kmax1 = tc_max_kp(e->dpad, nout, split, 1);
  const int kmax = k <= kmax2 ? kmax2 : kmax1;
  for (int64_t c0 = 0; c0 < k; c0 += kmax) {
    const int kc = (int)((k - c0) < kmax ? (k - c0) : kmax);
    const int kp = (kc + 15) / 16 * 16;
    const int lbm = peer_epoch ? 0 : tc_lb_mode(e->dpad, nout, split, kp);  // published tiles: classic layout
    const bool lb = lbm == 1 || lbm == 2;  // lbm 3 (W2) keeps the all-tf32 RHS tiles
    const int nab = lbm ? tc_lb_nab(lbm, kp) : (kp <= kmax2 ? 2 : 1);
    int rc = KGP_OK;
    if (!peer_epoch && !(skip_prep && kc == k)) {
      rc = e->bsplit.ensure((size_t)nblk * tc_rhs_block_bytes(split, lb, kp));
      if (rc) return rc;
      rc = prep_rhs(split, lb ? 1 : 0, e->n, k, c0, kp, b, b_rs, b_cs, e->bsplit.as<uint8_t>(), st,
                    cc ? cc->blk0 : 0, cc ? cc->blk1 : -1);
      if (rc) return rc;
    }
    TcParams p{};
    p.xrow = xrow;
    p.xcol = e->xcol.as<float>();
    p.bsplit = e->bsplit.as<uint8_t>();
    p.nrows = nrows;
    p.nblk = nblk;
    p.kp = kp;
    p.k = kc;
    p.nsa = tc_nsa(e->dpad, nout, split, kp);
    p.nab = nab;
    p.lb = lbm;
    const int nsplit = tc_col_chunk_splits(nrows, nblk);
    p.nper = (nblk + nsplit - 1) / nsplit;
    p.part = nullptr;
    if (cc) {  // one column chunk: its own split of [blk0, blk1), partials kept for the chunks after it
      KGP_REQUIRE(kc == k && !peer_epoch, KGP_ERR_STATE, "column-chunked product needs k in one launch");
      const int nb = cc->blk1 - cc->blk0;
      const int ns = tc_col_chunk_splits(nrows, nb);
      p.tbeg = cc->blk0;
      p.nblk = cc->blk1;
      p.nper = (nb + ns - 1) / ns;
      cc->used = (nb + p.nper - 1) / p.nper;
      KGP_REQUIRE(cc->slot0 + cc->used <= cc->slots_total, KGP_ERR_STATE, "column-chunk slots overrun");
      rc = e->tcpart.ensure(sizeof(float) * (size_t)cc->slots_total * nrows * nout * kp);
      if (rc) return rc;
      p.part = e->tcpart.as<float>();
      p.slot0 = cc->slot0;
      p.noreduce = cc->reduce ? 0 : 1;
    } else if (nsplit > 1) {
      rc = e->tcpart.ensure(sizeof(float) * (size_t)nsplit * nrows * nout * kp);
      if (rc) return rc;
      p.part = e->tcpart.as<float>();
    }
    p.flush = lbm == 3 ? tc_env_int("KGP_TC_W2FLUSH", 8) : tc_flush_blocks(nab);  // W2: one buffer, flush 8 (error)
    p.debug = tc_env_int("KGP_TC_DEBUG", 0);
    p.f2 = e->f * e->f;
    p.s = e->s;
    p.two_f = 2.0 * e->f;
    p.scale_dl = scale_dl_fast(e->kt, e->l, e->f);
    p.b = b + c0 * b_cs;
    p.b_rs = b_rs;
    p.b_cs = b_cs;
    p.diag_row0 = diag_row0;
    p.out_k = out_k ? out_k + c0 * o_cs : nullptr;
    p.out_dl = out_dl ? out_dl + c0 * o_cs : nullptr;
    p.out_df = out_df ? out_df + c0 * o_cs : nullptr;
    p.o_rs = o_rs;
    p.o_cs = o_cs;
    p.gate = e->gate;
    if (peer_epoch) {
      p.npeer = e->pworld;
      for (int q = 0; q < e->pworld; ++q) {
        p.pblk0[q] = (int)(e->prow[q] / 32);
        p.ptile[q] = e->pbase[q] + PEER_HDR;
        p.pready[q] = reinterpret_cast<const unsigned long long*>(e->pbase[q]);
      }
      p.pblk0[e->pworld] = nblk;
      p.epoch = peer_epoch;
      p.ptimeout_ns = e->ptimeout_ns;
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (e->timing && cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone) {
      if (e->tev_used + 2 > e->tev.size()) {
        for (int i = 0; i < 2; ++i) {
          cudaEvent_t ev;
          KGP_CUDA(cudaEventCreate(&ev));
          e->tev.push_back(ev);
        }
      }
      p.ev_start = e->tev[e->tev_used++];
      p.ev_stop = e->tev[e->tev_used++];
    }
    static const char* trace_path = getenv("KGP_TC_TRACE");  // diagnostic pipeline trace
    static unsigned long long* trace_buf = nullptr;
    if (trace_path && !trace_buf) KGP_CUDA(cudaMalloc(&trace_buf, 10 * 256 * sizeof(unsigned long long)));
    if (trace_path) {
      KGP_CUDA(cudaMemsetAsync(trace_buf, 0, 10 * 256 * sizeof(unsigned long long), st));
      p.trace = trace_buf;
    }
    rc = launch_kmm_tc(e->kt, e->dpad, nout, split, p, st);
    if (rc) return rc;
    if (trace_path) {
      unsigned long long h[10 * 256];
      KGP_CUDA(cudaMemcpyAsync(h, trace_buf, sizeof(h), cudaMemcpyDeviceToHost, st));
      KGP_CUDA(cudaStreamSynchronize(st));
      if (FILE* fh = fopen(trace_path, "ab")) {
        fwrite(h, sizeof(h), 1, fh);
        fclose(fh);
      }
    }
  }
  return KGP_OK;
}

// out[i, c] += dn[map[c]][row0 + i] * B[row0 + i, c]: the heteroscedastic part of the shift
__global__ void diag_shift_kernel(int64_t nrows, int64_t n, int64_t row0, const double* __restrict__ dn,
                                  const int32_t* __restrict__ map, const double* __restrict__ b, int64_t b_rs,
                                  int64_t b_cs, double* __restrict__ out, int64_t o_rs, int64_t o_cs) {
  const int c = blockIdx.y;
  const double* dc = dn + (int64_t)map[c] * n + row0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x)
    out[i * o_rs + c * o_cs] += dc[i] * b[(row0 + i) * b_rs + c * b_cs];
}

static int engine_matmul_core(kgp_engine_s* e, int64_t k, const double* b, int64_t b_rs, int64_t b_cs,
                              double* out_k, double* out_dl, double* out_df, int64_t o_rs, int64_t o_cs,
                              cudaStream_t st);

int engine_matmul_impl(kgp_engine_s* e, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* out_k,
                       double* out_dl, double* out_df, int64_t o_rs, int64_t o_cs, cudaStream_t st) {
  if (k <= 0 || e->nrows <= 0) return KGP_OK;
  if (!out_k && !out_dl && !out_df) return KGP_OK;
  KGP_REQUIRE(!(out_k && e->dn_classes > 0) || k <= e->dn_ncols, KGP_ERR_INVALID,
              "engine diagonal maps %lld columns, B has %lld", (long long)e->dn_ncols, (long long)k);
  int rc = engine_matmul_core(e, k, b, b_rs, b_cs, out_k, out_dl, out_df, o_rs, o_cs, st);
  if (rc || !out_k || e->dn_classes == 0) return rc;
  int64_t bx = (e->nrows + 255) / 256;
  if (bx > 256) bx = 256;
  diag_shift_kernel<<<dim3((unsigned)bx, (unsigned)k), 256, 0, st>>>(e->nrows, e->n, e->row0, e->dn.as<double>(),
                                                                    e->dmap.as<int32_t>(), b, b_rs, b_cs, out_k,
                                                                    o_rs, o_cs);
  KGP_LAUNCH("diag_shift_kernel");
  return KGP_OK;
}

__global__ void dense_finish_kernel(int64_t n, double f2, double s, double* k) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    double v = f2 * k[e];
    if (e / n == e % n) v += s;
    k[e] = v;
  }
}

// Khat = f^2 kappa(X, X) + s I, materialised once (kmat.py:107-123: the reference's DENSE
// mode, auto-selected for n <= 20000), through the parity panel kernel (numba's rounding)
static int dense_build(kgp_engine_s* e, cudaStream_t st) {
  if (e->dense_valid) return KGP_OK;
  int rc = e->dense.ensure(sizeof(double) * (size_t)e->n * e->n);
  if (rc) return rc;
  rc = kgp_eval_panel(e->kt, 0, e->n, e->n, e->d, e->x64.as<double>(), e->x64.as<double>(), e->l,
                      e->dense.as<double>(), e->n, st);
  if (rc) return rc;
  dense_finish_kernel<<<1184, 256, 0, st>>>(e->n, e->f * e->f, e->s, e->dense.as<double>());
  KGP_LAUNCH("dense_finish_kernel");
  // the packed upper triangle for products with <= SYM_MAXK columns (and its partial-sum
  // buffer, allocated here so no allocation happens inside a captured PCG graph)
  rc = e->dpack.ensure(sizeof(double) * (size_t)sym_packed_elems(e->n));
  if (rc) return rc;
  rc = e->dq.ensure(sizeof(double) * (size_t)sym_q_elems(e->n));
  if (rc) return rc;
  rc = sym_pack(e->n, e->dense.as<double>(), e->dpack.as<double>(), st);
  if (rc) return rc;
  if (!e->cublas) {
    cublasHandle_t h;
    KGP_REQUIRE(cublasCreate(&h) == CUBLAS_STATUS_SUCCESS, KGP_ERR_CUDA, "cublasCreate failed");
    e->cublas = h;
  }
  e->dense_valid = true;
  return KGP_OK;
}

static int engine_matmul_core(kgp_engine_s* e, int64_t k, const double* b, int64_t b_rs, int64_t b_cs,
                              double* out_k, double* out_dl, double* out_df, int64_t o_rs, int64_t o_cs,
                              cudaStream_t st) {
  if (e->precision == KGP_FP64 && e->dense_on && out_k && !out_dl && !out_df && b_rs == 1 && o_rs == 1 &&
      b_cs >= e->n && o_cs >= e->nrows) {
    // out (nrows x k, column-major) = Khat[row0:row0+nrows, :] B; Khat symmetric and row-major,
    // i.e. column-major Khat^T = Khat, so the row block is op(A) = A^T of column block row0.
    // (A hand-written DMMA m8n8k4 skinny kernel was measured against this cuBLAS call and
    // rejected: DESIGN.md, "DENSE-mode product".)
    int rc = dense_build(e, st);
    if (rc) return rc;
    // few columns on the full operator: the packed symmetric product (symv.cu; half the
    // bytes, L2-resident) -- env KGP_DENSE_SYM=0 keeps cuBLAS
    static const bool sym_on = [] {
      const char* s = getenv("KGP_DENSE_SYM");
      return !(s && atoi(s) == 0);
    }();
    if (sym_on && k <= SYM_MAXK && e->nrows == e->n && e->row0 == 0)
      return sym_matmul(e->n, e->dpack.as<double>(), (int)k, b, b_cs, out_k, o_cs, e->dq.as<double>(), st);
    cublasHandle_t h = (cublasHandle_t)e->cublas;
    KGP_REQUIRE(cublasSetStream(h, st) == CUBLAS_STATUS_SUCCESS, KGP_ERR_CUDA, "cublasSetStream failed");
    const double one = 1.0, zero = 0.0;
    const cublasStatus_t cs = cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)e->nrows, (int)k, (int)e->n, &one,
                                          e->dense.as<double>() + e->row0 * e->n, (int)e->n, b, (int)b_cs, &zero,
                                          out_k, (int)o_cs);
    KGP_REQUIRE(cs == CUBLAS_STATUS_SUCCESS, KGP_ERR_CUDA, "cublasDgemm failed (%d)", (int)cs);
    count_launches(1);
    return KGP_OK;
  }
  if (e->precision == KGP_FP64) {
    F64Params p{};
    p.gate = e->gate;
    p.xr = e->x64.as<double>() + e->row0 * e->d;
    p.xc = e->x64.as<double>();
    p.nrows = e->nrows;
    p.ncols = e->n;
    p.d = e->d;
    p.k = (int)k;
    p.l = e->l;
    p.f2 = e->f * e->f;
    p.s = e->s;
    p.two_f = 2.0 * e->f;
    p.f2_dl = e->f * e->f;
    p.b = b;
    p.b_rs = b_rs;
    p.b_cs = b_cs;
    p.diag_row0 = e->row0;
    p.out_k = out_k;
    p.out_dl = out_dl;
    p.out_df = out_df;
    p.o_rs = o_rs;
    p.o_cs = o_cs;
    return launch_kmm_f64(e->kt, p, e->f64part, st);
  }
  int rc = engine_prepare(e, st);
  if (rc) return rc;
  return tc_matmul(e, e->xrow.as<float>(), e->nrows, e->row0, k, b, b_rs, b_cs, out_k, out_dl, out_df, o_rs, o_cs,
                   st);
}

}  // namespace kgp

using namespace kgp;

#define CHECK_ENGINE(e)                                                                          \
  KGP_REQUIRE((e) != nullptr && handle_live(e) && (e)->magic == ENGINE_MAGIC, KGP_ERR_STATE, \
              "invalid or destroyed engine handle")
#define CHECK_PRECOND(p)                                                                          \
  KGP_REQUIRE((p) != nullptr && handle_live(p) && (p)->magic == PRECOND_MAGIC, KGP_ERR_STATE, \
              "invalid or destroyed preconditioner handle")

extern "C" int kgp_version(void) { return KGP_ABI_VERSION; }

extern "C" int64_t kgp_launch_count(void) { return g_launches.load(); }

extern "C" int kgp_engine_set_timing(kgp_engine* e, int enable) {
  CHECK_ENGINE(e);
  e->timing = enable != 0;
  e->tev_used = 0;
  return KGP_OK;
}

extern "C" int kgp_engine_kernel_time(kgp_engine* e, double* ms, int64_t* launches) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(ms != nullptr && launches != nullptr, KGP_ERR_INVALID, "output pointer is NULL");
  double total = 0.0;
  for (size_t i = 0; i + 1 < e->tev_used; i += 2) {
    KGP_CUDA(cudaEventSynchronize(e->tev[i + 1]));
    float t = 0.f;
    KGP_CUDA(cudaEventElapsedTime(&t, e->tev[i], e->tev[i + 1]));
    total += t;
  }
  *ms = total;
  *launches = (int64_t)(e->tev_used / 2);
  e->tev_used = 0;
  return KGP_OK;
}

extern "C" const char* kgp_last_error(void) { return g_err_msg; }

extern "C" int kgp_device_count(int* count) {
  KGP_REQUIRE(count != nullptr, KGP_ERR_INVALID, "count pointer is NULL");
  KGP_CUDA(cudaGetDeviceCount(count));
  return KGP_OK;
}

static int check_params(double l, double f, double s) {
  KGP_REQUIRE(l > 0.0 && l < INFINITY, KGP_ERR_INVALID, "hyperparameter l must be positive and finite, got %g", l);
  KGP_REQUIRE(f > 0.0 && f < INFINITY, KGP_ERR_INVALID, "hyperparameter f must be positive and finite, got %g", f);
  KGP_REQUIRE(s > 0.0 && s < INFINITY, KGP_ERR_INVALID, "hyperparameter s must be positive and finite, got %g", s);
  return KGP_OK;
}

extern "C" int kgp_engine_create(kgp_engine** out, int device, int kernel, int precision, int64_t n, int d,
                                 const double* x, int x_on_device, double l, double f, double s, void* stream) {
  KGP_REQUIRE(out != nullptr, KGP_ERR_INVALID, "out pointer is NULL");
  *out = nullptr;
  KGP_REQUIRE(kernel >= 0 && kernel <= 2, KGP_ERR_INVALID, "unknown kernel id %d", kernel);
  KGP_REQUIRE(precision >= 0 && precision <= 3, KGP_ERR_INVALID, "unknown precision %d", precision);
  KGP_REQUIRE(n >= 1 && d >= 1, KGP_ERR_INVALID, "X must be a nonempty 2-d array, got (%lld, %d)", (long long)n, d);
  KGP_REQUIRE(d <= 16, KGP_ERR_INVALID, "dimension d=%d exceeds the supported maximum of 16", d);
  KGP_REQUIRE(x != nullptr, KGP_ERR_INVALID, "X pointer is NULL");
  int rc = check_params(l, f, s);
  if (rc) return rc;
  KGP_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  kgp_engine_s* e = new kgp_engine_s();
  e->magic = ENGINE_MAGIC;
  e->device = device;
  e->kt = kernel;
  e->precision = precision;
  e->n = n;
  e->d = d;
  e->dpad = tc_pad_dim(d);
  e->row0 = 0;
  e->nrows = n;
  e->l = l;
  e->f = f;
  e->s = s;
  e->prepared = false;
  e->hstatus = nullptr;
  rc = cuda_check(cudaMallocHost(&e->hstatus, sizeof(int32_t) * 4), "pinned status");
  for (int i = 0; i < PCG_LOOKAHEAD && !rc; ++i)
    rc = cuda_check(cudaEventCreateWithFlags(&e->events[i], cudaEventDisableTiming), "event create");
  if (!rc) rc = cuda_check(cudaStreamCreateWithFlags(&e->cstream, cudaStreamNonBlocking), "stream create");
  if (!rc) rc = e->x64.ensure(sizeof(double) * n * d);
  if (!rc) rc = e->mean.ensure(sizeof(double) * d);
  if (!rc)
    rc = cuda_check(cudaMemcpyAsync(e->x64.p, x, sizeof(double) * n * d,
                                    x_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st),
                    "copy X");
  if (!rc) rc = col_mean(n, d, e->x64.as<double>(), e->mean.as<double>(), st);
  if (!rc && !x_on_device) rc = cuda_check(cudaStreamSynchronize(st), "engine create");
  if (rc) {
    engine_free_host_state(e);
    delete e;
    return rc;
  }
  {
    std::lock_guard<std::mutex> g(g_handles_mu);
    g_handles.insert(e);
  }
  *out = e;
  return KGP_OK;
}

extern "C" int kgp_engine_set_params(kgp_engine* e, double l, double f, double s, void* stream) {
  CHECK_ENGINE(e);
  int rc = check_params(l, f, s);
  if (rc) return rc;
  if (l != e->l) e->prepared = false;
  if (l != e->l || f != e->f || s != e->s) e->dense_valid = false;
  if (l != e->l || f != e->f || s != e->s) bump_graph_epoch();
  e->l = l;
  e->f = f;
  e->s = s;
  (void)stream;
  return KGP_OK;
}

extern "C" int kgp_engine_set_precision(kgp_engine* e, int precision) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(precision >= 0 && precision <= 3, KGP_ERR_INVALID, "unknown precision %d", precision);
  e->precision = precision;
  e->prepared = false;
  bump_graph_epoch();
  return KGP_OK;
}

extern "C" int kgp_engine_set_rows(kgp_engine* e, int64_t row0, int64_t nrows) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(row0 >= 0 && nrows >= 0 && row0 + nrows <= e->n, KGP_ERR_INVALID, "row range [%lld, %lld) outside [0, %lld)",
              (long long)row0, (long long)(row0 + nrows), (long long)e->n);
  e->row0 = row0;
  e->nrows = nrows;
  e->prepared = false;
  bump_graph_epoch();
  return KGP_OK;
}

extern "C" int kgp_engine_set_dense(kgp_engine* e, int enable) {
  CHECK_ENGINE(e);
  const bool on = enable != 0;
  if (on != e->dense_on) bump_graph_epoch();
  e->dense_on = on;
  if (!on) {
    e->dense.release();
    e->dense_valid = false;
  }
  return KGP_OK;
}

extern "C" int kgp_engine_set_diag(kgp_engine* e, int classes, const double* dn, int64_t ncols, const int32_t* map,
                                   void* stream) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(classes >= 0, KGP_ERR_INVALID, "classes must be >= 0");
  bump_graph_epoch();
  if (classes == 0) {
    e->dn_classes = 0;
    e->dn_ncols = 0;
    return KGP_OK;
  }
  KGP_REQUIRE(dn != nullptr && map != nullptr && ncols >= 1, KGP_ERR_INVALID, "NULL diagonal or column map");
  for (int64_t c = 0; c < ncols; ++c)
    KGP_REQUIRE(map[c] >= 0 && map[c] < classes, KGP_ERR_INVALID, "column %lld maps to class %d of %d",
                (long long)c, map[c], classes);
  KGP_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = e->dn.ensure(sizeof(double) * (size_t)classes * e->n);
  if (!rc) rc = e->dmap.ensure(sizeof(int32_t) * (size_t)ncols);
  if (rc) return rc;
  KGP_CUDA(cudaMemcpyAsync(e->dn.p, dn, sizeof(double) * (size_t)classes * e->n, cudaMemcpyDeviceToDevice, st));
  KGP_CUDA(cudaMemcpyAsync(e->dmap.p, map, sizeof(int32_t) * (size_t)ncols, cudaMemcpyHostToDevice, st));
  KGP_CUDA(cudaStreamSynchronize(st));
  e->dn_classes = classes;
  e->dn_ncols = ncols;
  return KGP_OK;
}

extern "C" int kgp_engine_destroy(kgp_engine* e) {
  {
    std::lock_guard<std::mutex> g(g_handles_mu);
    if (e == nullptr || g_handles.count(e) == 0) {
      set_error(KGP_ERR_STATE, "engine handle already destroyed or never created");
      return KGP_ERR_STATE;
    }
    g_handles.erase(e);
  }
  cudaSetDevice(e->device);
  cudaDeviceSynchronize();
  e->magic = DEAD_MAGIC;
  engine_free_host_state(e);
  delete e;
  return KGP_OK;
}

extern "C" int kgp_engine_matmul(kgp_engine* e, int64_t k, const double* b, int64_t b_rs, int64_t b_cs, double* out_k,
                                 double* out_dl, double* out_df, int64_t o_rs, int64_t o_cs, void* stream) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(k >= 1, KGP_ERR_INVALID, "B must have at least one column");
  KGP_REQUIRE(b != nullptr, KGP_ERR_INVALID, "B pointer is NULL");
  KGP_CUDA(cudaSetDevice(e->device));
  return engine_matmul_impl(e, k, b, b_rs, b_cs, out_k, out_dl, out_df, o_rs, o_cs, (cudaStream_t)stream);
}

// Host-buffer product with the device->host transfer of the outputs pipelined behind the
// computation: rows are processed in chunks, each chunk's outputs copied back on the
// engine's copy stream while the next chunk computes. Returns when the host outputs hold
// the result.
extern "C" int kgp_engine_matmul_host(kgp_engine* e, int64_t k, const double* b, double* out_k, double* out_dl,
                                      double* out_df, void* stream) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(k >= 1 && b != nullptr, KGP_ERR_INVALID, "B must be a non-NULL host array with >= 1 column");
  KGP_REQUIRE(out_k || out_dl || out_df, KGP_ERR_INVALID, "no output requested");
  KGP_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = e->n, rows = e->nrows;
  const int nout = (out_k ? 1 : 0) + (out_dl ? 1 : 0) + (out_df ? 1 : 0);
  int rc = e->hostbuf.ensure(sizeof(double) * (size_t)k * (n + nout * rows));
  if (rc) return rc;
  double* db = e->hostbuf.as<double>();
  double* dout = db + k * n;
  double* dk = out_k ? dout : nullptr;
  double* dl = out_dl ? dout + (out_k ? 1 : 0) * rows * k : nullptr;
  double* df = out_df ? dout + (nout - 1) * rows * k : nullptr;
  // chunk only the tensor-core path without a heteroscedastic diagonal, when k fits one launch
  const int split = tc_split_of(e->precision);
  const bool chunked = e->precision != KGP_FP64 && e->dn_classes == 0 &&
                       k <= tc_max_kp(e->dpad, out_dl ? 2 : 1, split, 1) && rows >= 32768;
  if (!e->xstream) {
    KGP_CUDA(cudaStreamCreateWithFlags(&e->xstream, cudaStreamNonBlocking));
    for (auto& ev : e->xev) KGP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : e->zev) KGP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  // input pipelining (chunked path): B's rows are the operator's COLUMNS, so the first row chunk
  // runs as nz column-chunked launches, launch c needing only B's rows of column chunk c -- the
  // host->device copy of chunk c + 1 (copy stream) overlaps launch c; every later row chunk
  // finds all of B resident (KGP_HOST_ZCHUNKS, default 3; 1 = one copy before any compute)
  const int64_t nblk_all = (n + 31) / 32;
  // Chunk sizes grow geometrically (ratio KGP_HOST_ZRATIO, default 4; 3 chunks: 1/21, 4/21 and
  // 16/21 of B): only the first, small copy is exposed, and launch c (chunk c's columns for ~40 %
  // of the rows) outlasts the copy of chunk c + 1 (tools/e2e_zchunks.sh: cfg2 e2e 3.50 -> 3.27 ms)
  int nz = chunked ? tc_env_int("KGP_HOST_ZCHUNKS", 3) : 1;
  nz = nz < 1 ? 1 : (nz > 8 ? 8 : nz);
  if (nz > nblk_all) nz = (int)nblk_all;
  const double zr = std::max(1.0, tc_env_int("KGP_HOST_ZRATIO", 4) / 1.0);
  auto zblk = [&](int c) -> int {
    if (c <= 0) return 0;
    if (c >= nz) return (int)nblk_all;
    const double f = zr == 1.0 ? (double)c / nz : (std::pow(zr, c) - 1.0) / (std::pow(zr, nz) - 1.0);
    return (int)std::max<int64_t>(c, std::min<int64_t>(nblk_all - (nz - c), (int64_t)(f * nblk_all + 0.5)));
  };
  if (nz > 1) {
    KGP_CUDA(cudaEventRecord(e->zev[8], st));  // the copy stream starts after earlier work on st
    KGP_CUDA(cudaStreamWaitEvent(e->xstream, e->zev[8], 0));
    for (int c = 0; c < nz; ++c) {
      const int64_t j0 = (int64_t)zblk(c) * 32, j1 = std::min<int64_t>(n, (int64_t)zblk(c + 1) * 32);
      KGP_CUDA(cudaMemcpyAsync(db + j0 * k, b + j0 * k, sizeof(double) * (j1 - j0) * k, cudaMemcpyHostToDevice,
                               e->xstream));
      KGP_CUDA(cudaEventRecord(e->zev[c], e->xstream));
    }
  } else {
    KGP_CUDA(cudaMemcpyAsync(db, b, sizeof(double) * n * k, cudaMemcpyHostToDevice, st));
  }
  // Row chunks shrinking geometrically (KGP_HOST_CHUNKS = 3, share ratio KGP_HOST_RRATIO = 50 %:
  // ~4/7, 2/7, 1/7 of the rows) with every boundary snapped to whole waves of 148 row tiles: each
  // chunk's output copy hides behind the chunks after it, only the last, small chunk's copy is
  // exposed. cfg2 (tools/e2e_tail4.sh, KGP_HOST_TRACE=1 timelines): 3.14 ms. Without the wave
  // snapping the same ratios gave 3.14-3.65 ms -- a chunk of 276 or 310 row tiles runs 2 partial
  // waves (the column split cannot refill them at the small input chunks). KGP_HOST_RRATIO=0: the
  // earlier schedule, equal shares with the last one KGP_HOST_TAIL percent of a share (3.28 ms)
  const int max_chunks = (int)(sizeof(e->xev) / sizeof(e->xev[0]));
  int nchunk = chunked ? tc_env_int("KGP_HOST_CHUNKS", KGP_HOST_CHUNKS_DEFAULT) : 1;
  nchunk = nchunk < 1 ? 1 : (nchunk > max_chunks ? max_chunks : nchunk);
  if (chunked) {
    rc = engine_prepare(e, st);
    if (rc) return rc;
  }
  double* hosts[3] = {out_k, out_dl, out_df};
  double* devs[3] = {dk, dl, df};
  const bool trace = tc_env_int("KGP_HOST_TRACE", 0) != 0;
  cudaEvent_t tev[1 + 2 * 8] = {};
  if (trace) {
    for (auto& ev : tev) KGP_CUDA(cudaEventCreate(&ev));
    KGP_CUDA(cudaEventRecord(tev[0], st));  // after the input copies were queued (they run on the copy stream)
  }
  // chunk boundaries on 128-row CTA tiles
  const int64_t blocks = (rows + 127) / 128;
  std::vector<int64_t> edges(nchunk + 1, 0);
  {
    const double q = tc_env_int("KGP_HOST_RRATIO", KGP_HOST_RRATIO_DEFAULT) / 100.0;
    const bool waves = tc_env_int("KGP_HOST_WAVES", 1) != 0;
    edges[nchunk] = blocks;
    for (int c = 1; c < nchunk; ++c) {
      int64_t t;
      if (q > 0.0 && q != 1.0) {
        // geometric shares; each boundary snapped to whole waves of 148 row tiles past the previous
        // one (a launch over whole waves needs no column split to fill the SMs)
        const double target = (1.0 - std::pow(q, c)) / (1.0 - std::pow(q, nchunk)) * (double)blocks;
        t = waves ? edges[c - 1] + std::max<int64_t>(1, (int64_t)((target - (double)edges[c - 1]) / 148.0 + 0.5)) * 148
                  : (int64_t)(target + 0.5);
      } else {
        // equal shares, the last one KGP_HOST_TAIL percent of a share
        const double tail = tc_env_int("KGP_HOST_TAIL", 35) / 100.0;
        const double last = tail / (nchunk - 1 + tail);
        t = (int64_t)((double)c * (1.0 - last) / (nchunk - 1) * (double)blocks + 0.5);
      }
      edges[c] = std::max(edges[c - 1] + 1, std::min(t, blocks - (nchunk - c)));
    }
  }
  for (int c = 0; c < nchunk; ++c) {
    auto edge = [&](int c2) -> int64_t { return std::min(rows, edges[c2] * 128); };
    const int64_t r0 = edge(c), r1 = edge(c + 1);
    if (r1 <= r0) continue;
    if (chunked && c == 0 && nz > 1) {
      int total = 0;  // partial slots over all column chunks (tc_matmul's split of each chunk)
      for (int z = 0; z < nz; ++z) {
        const int nb = zblk(z + 1) - zblk(z);
        const int ns = tc_col_chunk_splits(r1 - r0, nb), nper = (nb + ns - 1) / ns;
        total += (nb + nper - 1) / nper;
      }
      int slot = 0;
      for (int z = 0; z < nz && !rc; ++z) {
        KGP_CUDA(cudaStreamWaitEvent(st, e->zev[z], 0));
        ColChunk cc{zblk(z), zblk(z + 1), slot, total, z == nz - 1, 0};
        rc = tc_matmul(e, e->xrow.as<float>() + r0 * (e->dpad + 1), r1 - r0, e->row0 + r0, k, db, k, 1,
                       dk ? dk + r0 * k : nullptr, dl ? dl + r0 * k : nullptr, df ? df + r0 * k : nullptr, k, 1,
                       st, false, 0, &cc);
        slot += cc.used;
      }
    } else if (chunked) {
      rc = tc_matmul(e, e->xrow.as<float>() + r0 * (e->dpad + 1), r1 - r0, e->row0 + r0, k, db, k, 1,
                     dk ? dk + r0 * k : nullptr, dl ? dl + r0 * k : nullptr, df ? df + r0 * k : nullptr, k, 1, st,
                     c > 0);
    } else {
      rc = engine_matmul_impl(e, k, db, k, 1, dk, dl, df, k, 1, st);
    }
    if (rc) return rc;
    KGP_CUDA(cudaEventRecord(e->xev[c], st));
    if (trace) KGP_CUDA(cudaEventRecord(tev[1 + 2 * c], st));
    KGP_CUDA(cudaStreamWaitEvent(e->xstream, e->xev[c], 0));
    for (int o = 0; o < 3; ++o)
      if (hosts[o])
        KGP_CUDA(cudaMemcpyAsync(hosts[o] + r0 * k, devs[o] + r0 * k, sizeof(double) * (r1 - r0) * k,
                                 cudaMemcpyDeviceToHost, e->xstream));
    if (trace) KGP_CUDA(cudaEventRecord(tev[2 + 2 * c], e->xstream));
  }
  KGP_CUDA(cudaStreamSynchronize(e->xstream));
  if (trace) {  // diagnostic timeline (KGP_HOST_TRACE=1): per row chunk, compute done / copy done (us)
    fprintf(stderr, "kgp host trace (rows %lld, %d chunks, %d input chunks):", (long long)rows, nchunk, nz);
    for (int c = 0; c < nchunk; ++c) {
      float a = 0.f, b2 = 0.f;
      cudaEventElapsedTime(&a, tev[0], tev[1 + 2 * c]);
      cudaEventElapsedTime(&b2, tev[0], tev[2 + 2 * c]);
      fprintf(stderr, " [%d: compute %.0f, copy %.0f]", c, a * 1e3f, b2 * 1e3f);
    }
    fprintf(stderr, "\n");
    for (auto ev : tev) cudaEventDestroy(ev);
  }
  return KGP_OK;
}

extern "C" int kgp_engine_cross_matmul(kgp_engine* e, int64_t m, const double* xs, int64_t k, const double* b,
                                       int64_t b_rs, int64_t b_cs, double* out, int64_t o_rs, int64_t o_cs,
                                       void* stream) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(k >= 1 && m >= 0, KGP_ERR_INVALID, "bad cross shape");
  if (m == 0) return KGP_OK;
  KGP_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (e->precision == KGP_FP64) {
    F64Params p{};
    p.xr = xs;
    p.xc = e->x64.as<double>();
    p.nrows = m;
    p.ncols = e->n;
    p.d = e->d;
    p.k = (int)k;
    p.l = e->l;
    p.f2 = e->f * e->f;
    p.s = 0.0;
    p.two_f = 0.0;
    p.f2_dl = 0.0;
    p.b = b;
    p.b_rs = b_rs;
    p.b_cs = b_cs;
    p.diag_row0 = -1;
    p.out_k = out;
    p.o_rs = o_rs;
    p.o_cs = o_cs;
    return launch_kmm_f64(e->kt, p, e->f64part, st);
  }
  int rc = engine_prepare(e, st);
  if (rc) return rc;
  rc = e->xrow_cross.ensure(sizeof(float) * (size_t)(m + 1) * (e->dpad + 1));
  if (rc) return rc;
  rc = prep_rows(e->kt, 0, e->d, e->dpad, m, xs, e->mean.as<double>(), e->l, e->xrow_cross.as<float>(), st);
  if (rc) return rc;
  return tc_matmul(e, e->xrow_cross.as<float>(), m, -1, k, b, b_rs, b_cs, out, nullptr, nullptr, o_rs, o_cs, st);
}

// ------------------------------------------------------------------ preconditioner
extern "C" int kgp_precond_create(kgp_precond** out, int64_t n, int64_t m, const double* wt, double s, void* stream) {
  KGP_REQUIRE(out != nullptr && wt != nullptr, KGP_ERR_INVALID, "NULL pointer");
  KGP_REQUIRE(n >= 1 && m >= 1 && m <= n, KGP_ERR_INVALID, "need 1 <= m <= n, got m=%lld, n=%lld", (long long)m,
              (long long)n);
  KGP_REQUIRE(s > 0.0, KGP_ERR_INVALID, "shift must be positive");
  kgp_precond_s* p = new kgp_precond_s();
  p->magic = PRECOND_MAGIC;
  p->kind = KGP_PRECOND_NYSTROM;
  p->n = n;
  p->m = m;
  p->s = s;
  int rc = p->wt.ensure(sizeof(double) * n * m);
  if (!rc)
    rc = cuda_check(cudaMemcpyAsync(p->wt.p, wt, sizeof(double) * n * m, cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
                    "copy W");
  if (rc) {
    delete p;
    return rc;
  }
  {
    std::lock_guard<std::mutex> g(g_handles_mu);
    g_handles.insert(p);
  }
  *out = p;
  return KGP_OK;
}

extern "C" int kgp_afn_create(kgp_precond** out, int64_t n, int64_t m, const int64_t* perm, const double* linv,
                              const double* l11, const double* w, int npt1, const double* gval, const int32_t* gcol,
                              int64_t nnz, const int32_t* gtptr, const int32_t* gtrow, const double* gtval, double s,
                              void* stream) {
  KGP_REQUIRE(out != nullptr && perm != nullptr && linv != nullptr && w != nullptr && gval != nullptr &&
                  gcol != nullptr && gtptr != nullptr && gtrow != nullptr && gtval != nullptr,
              KGP_ERR_INVALID, "NULL pointer");
  KGP_REQUIRE(n >= 2 && m >= 1 && m < n && n - m < ((int64_t)1 << 31), KGP_ERR_INVALID,
              "need 1 <= m < n, got m=%lld, n=%lld", (long long)m, (long long)n);
  KGP_REQUIRE(npt1 >= 1 && nnz >= n - m && nnz <= (int64_t)npt1 * (n - m), KGP_ERR_INVALID,
              "bad FSAI factor shape (npt1=%d, nnz=%lld)", npt1, (long long)nnz);
  KGP_REQUIRE(s > 0.0, KGP_ERR_INVALID, "shift must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  kgp_precond_s* p = new kgp_precond_s();
  p->magic = PRECOND_MAGIC;
  p->kind = KGP_PRECOND_AFN;
  p->n = n;
  p->m = m;
  p->s = s;
  p->n2 = n - m;
  p->npt1 = npt1;
  p->nnz = nnz;
  const int64_t n2 = n - m;
  struct Copy { DevBuf* dst; const void* src; size_t bytes; };
  const Copy copies[] = {
      {&p->perm, perm, sizeof(int64_t) * n},           {&p->linv, linv, sizeof(double) * m * m},
      {&p->w, w, sizeof(double) * n2 * m},             {&p->gval, gval, sizeof(double) * npt1 * n2},
      {&p->gcol, gcol, sizeof(int32_t) * npt1 * n2},   {&p->gtptr, gtptr, sizeof(int32_t) * (n2 + 1)},
      {&p->gtrow, gtrow, sizeof(int32_t) * nnz},       {&p->gtval, gtval, sizeof(double) * nnz}};
  int rc = KGP_OK;
  for (const Copy& c : copies) {
    rc = c.dst->ensure(c.bytes);
    if (!rc) rc = cuda_check(cudaMemcpyAsync(c.dst->p, c.src, c.bytes, cudaMemcpyDeviceToDevice, st), "copy AFN factor");
    if (rc) break;
  }
  if (!rc && l11) {
    rc = p->l11.ensure(sizeof(double) * m * m);
    if (!rc) rc = cuda_check(cudaMemcpyAsync(p->l11.p, l11, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st),
                             "copy AFN factor");
  }
  if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "AFN create");
  if (rc) {
    delete p;
    return rc;
  }
  {
    std::lock_guard<std::mutex> g(g_handles_mu);
    g_handles.insert(p);
  }
  *out = p;
  return KGP_OK;
}

extern "C" int kgp_precond_kind(kgp_precond* p, int* kind) {
  CHECK_PRECOND(p);
  KGP_REQUIRE(kind != nullptr, KGP_ERR_INVALID, "NULL pointer");
  *kind = p->kind;
  return KGP_OK;
}

extern "C" int kgp_precond_destroy(kgp_precond* p) {
  {
    std::lock_guard<std::mutex> g(g_handles_mu);
    if (p == nullptr || g_handles.count(p) == 0) {
      set_error(KGP_ERR_STATE, "preconditioner handle already destroyed or never created");
      return KGP_ERR_STATE;
    }
    g_handles.erase(p);
  }
  cudaDeviceSynchronize();
  p->magic = DEAD_MAGIC;
  delete p;
  return KGP_OK;
}

extern "C" int kgp_precond_apply_inverse(kgp_precond* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs,
                                         double* out, int64_t o_rs, int64_t o_cs, void* stream) {
  CHECK_PRECOND(p);
  KGP_REQUIRE(k >= 1, KGP_ERR_INVALID, "B must have at least one column");
  return precond_apply_impl(p, k, b, b_rs, b_cs, out, o_rs, o_cs, (cudaStream_t)stream);
}

extern "C" int kgp_lowrank_apply(kgp_precond* p, double beta, double alpha, int64_t k, const double* b, int64_t b_rs,
                                 int64_t b_cs, double* out, int64_t o_rs, int64_t o_cs, void* stream) {
  CHECK_PRECOND(p);
  KGP_REQUIRE(p->kind == KGP_PRECOND_NYSTROM, KGP_ERR_INVALID, "low-rank operations need a Nystrom handle");
  KGP_REQUIRE(k >= 1, KGP_ERR_INVALID, "B must have at least one column");
  return lowrank_apply_impl(p, beta, alpha, k, b, b_rs, b_cs, out, o_rs, o_cs, (cudaStream_t)stream);
}

extern "C" int kgp_lowrank_project(kgp_precond* p, int64_t k, const double* b, int64_t b_rs, int64_t b_cs,
                                   double* t_out, void* stream) {
  CHECK_PRECOND(p);
  KGP_REQUIRE(p->kind == KGP_PRECOND_NYSTROM, KGP_ERR_INVALID, "low-rank operations need a Nystrom handle");
  KGP_REQUIRE(k >= 1 && t_out != nullptr, KGP_ERR_INVALID, "bad projection arguments");
  return lowrank_project_impl(p, k, b, b_rs, b_cs, t_out, (cudaStream_t)stream);
}

extern "C" int kgp_lowrank_expand(kgp_precond* p, double beta, double alpha, int64_t k, const double* b, int64_t b_rs,
                                  int64_t b_cs, const double* t, double* out, int64_t o_rs, int64_t o_cs,
                                  void* stream) {
  CHECK_PRECOND(p);
  KGP_REQUIRE(p->kind == KGP_PRECOND_NYSTROM, KGP_ERR_INVALID, "low-rank operations need a Nystrom handle");
  KGP_REQUIRE(k >= 1 && t != nullptr, KGP_ERR_INVALID, "bad expansion arguments");
  return lowrank_expand_impl(p, beta, alpha, k, b, b_rs, b_cs, t, out, o_rs, o_cs, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ solvers
extern "C" int kgp_pcg(kgp_engine* e, kgp_precond* p, int64_t k, const double* y, double tol, int32_t max_iter,
                       double* x_out, double* alphas, double* betas, int32_t* iters, double* rel, int32_t* converged,
                       void* stream) {
  CHECK_ENGINE(e);
  if (p) CHECK_PRECOND(p);
  KGP_REQUIRE(tol >= 0.0 && max_iter >= 1, KGP_ERR_INVALID, "need tol >= 0 and max_iter >= 1");
  KGP_REQUIRE(e->row0 == 0 && e->nrows == e->n, KGP_ERR_INVALID, "kgp_pcg needs an unpartitioned engine");
  KGP_REQUIRE(!p || p->n == e->n, KGP_ERR_INVALID, "preconditioner size mismatch");
  KGP_CUDA(cudaSetDevice(e->device));
  return pcg_solve_impl(e, p, k, y, tol, max_iter, x_out, alphas, betas, iters, rel, converged, (cudaStream_t)stream);
}

extern "C" int kgp_slq_logdet(int64_t k, int32_t max_iter, const double* alphas, const double* betas,
                              const int32_t* iters, const double* norms_sq, double* logdet, void* stream) {
  KGP_REQUIRE(k >= 1, KGP_ERR_INVALID, "need at least one probe trace");
  KGP_REQUIRE(logdet != nullptr, KGP_ERR_INVALID, "logdet pointer is NULL");
  return slq_impl(k, max_iter, alphas, betas, iters, norms_sq, logdet, (cudaStream_t)stream);
}


// ------------------------------------------------------------------ fused all-gather + operator
namespace {

__global__ void peer_wait_done_kernel(int world, int rank, unsigned long long want, unsigned long long timeout_ns,
                                      const unsigned long long* f0, const unsigned long long* f1,
                                      const unsigned long long* f2, const unsigned long long* f3,
                                      const unsigned long long* f4, const unsigned long long* f5,
                                      const unsigned long long* f6, const unsigned long long* f7) {
  const unsigned long long* f[8] = {f0, f1, f2, f3, f4, f5, f6, f7};
  const int q = threadIdx.x;
  if (q < world && q != rank) kgp::peer_wait_flag(f[q], want, timeout_ns);
}

__global__ void peer_flag_kernel(unsigned long long* flag, unsigned long long v) { kgp::peer_set_flag(flag, v); }

}  // namespace

extern "C" int kgp_peer_alloc(int64_t bytes, void** dptr, void* ipc_handle) {
  KGP_REQUIRE(bytes > 0 && dptr != nullptr, KGP_ERR_INVALID, "bad peer buffer request");
  void* p = nullptr;
  KGP_CUDA(cudaMalloc(&p, (size_t)bytes));
  KGP_CUDA(cudaMemset(p, 0, PEER_HDR));  // flags start at 0 (no epoch published or read)
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    const cudaError_t rc = cudaIpcGetMemHandle(&h, p);
    if (rc != cudaSuccess) {
      cudaFree(p);
      return cuda_check(rc, "cudaIpcGetMemHandle");
    }
    memcpy(ipc_handle, &h, sizeof(h));
  }
  *dptr = p;
  return KGP_OK;
}

extern "C" int kgp_peer_open(const void* ipc_handle, void** dptr) {
  KGP_REQUIRE(ipc_handle != nullptr && dptr != nullptr, KGP_ERR_INVALID, "NULL handle");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  KGP_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return KGP_OK;
}

extern "C" int kgp_peer_close(void* dptr) {
  KGP_CUDA(cudaIpcCloseMemHandle(dptr));
  return KGP_OK;
}

extern "C" int kgp_peer_free(void* dptr) {
  KGP_CUDA(cudaFree(dptr));
  return KGP_OK;
}

extern "C" int kgp_engine_peer_buffer_bytes(kgp_engine* e, int64_t k, int64_t own_rows, int64_t* bytes) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(bytes != nullptr && k >= 1 && own_rows >= 0, KGP_ERR_INVALID, "bad peer buffer query");
  const int split = tc_split_of(e->precision);
  const int64_t kp = (k + 15) / 16 * 16;
  *bytes = PEER_HDR + (own_rows + 31) / 32 * (int64_t)tc_rhs_block_bytes(split, false, (int)kp);
  return KGP_OK;
}

// A peer configuration is valid only for the precision and row block it was set up with
// (tile sizes and block ownership depend on both); later set_precision / set_rows calls
// invalidate it, and publish / peer_matmul re-check before touching the shared buffers.
static int peer_check(const kgp_engine* e) {
  KGP_REQUIRE(e->pworld > 0, KGP_ERR_STATE, "no peer configuration (kgp_engine_set_peers)");
  KGP_REQUIRE(e->precision == e->pprec && e->precision != KGP_FP64, KGP_ERR_STATE,
              "engine precision changed since kgp_engine_set_peers (call it again)");
  KGP_REQUIRE(e->row0 == e->prow[e->prank] && e->nrows == e->prow[e->prank + 1] - e->prow[e->prank], KGP_ERR_STATE,
              "engine rows changed since kgp_engine_set_peers (call it again)");
  return KGP_OK;
}

extern "C" int kgp_engine_set_peers(kgp_engine* e, int world, int rank, const int64_t* row_start,
                                    void* const* bases, int64_t k_cap) {
  CHECK_ENGINE(e);
  KGP_REQUIRE(e->precision != KGP_FP64, KGP_ERR_INVALID, "the fused all-gather operator needs the tensor-core "
              "precision (fast or tf32)");
  KGP_REQUIRE(world >= 1 && world <= KGP_MAX_PEERS && rank >= 0 && rank < world && row_start && bases,
              KGP_ERR_INVALID, "bad peer configuration (world %d, rank %d; at most %d ranks)", world, rank,
              KGP_MAX_PEERS);
  KGP_REQUIRE(row_start[0] == 0 && row_start[world] == e->n, KGP_ERR_INVALID, "row blocks must cover [0, %lld)",
              (long long)e->n);
  for (int q = 0; q < world; ++q) {
    KGP_REQUIRE(row_start[q + 1] >= row_start[q] && (q + 1 == world || row_start[q + 1] % 32 == 0),
                KGP_ERR_INVALID, "row block boundaries must ascend on multiples of 32 (column blocks)");
    KGP_REQUIRE(bases[q] != nullptr, KGP_ERR_INVALID, "NULL peer buffer for rank %d", q);
  }
  KGP_REQUIRE(e->row0 == row_start[rank] && e->nrows == row_start[rank + 1] - row_start[rank], KGP_ERR_INVALID,
              "engine rows [%lld, %lld) are not rank %d's block [%lld, %lld) (kgp_engine_set_rows first)",
              (long long)e->row0, (long long)(e->row0 + e->nrows), rank, (long long)row_start[rank],
              (long long)row_start[rank + 1]);
  KGP_REQUIRE(k_cap >= 1, KGP_ERR_INVALID, "k_cap must be >= 1");
  e->pworld = world;
  e->prank = rank;
  e->pprec = e->precision;
  e->pkcap = k_cap;
  {
    // Peer waits trap after this long (a trapped context is lost for the process: size it
    // well above any host-side skew between ranks). KGP_PEER_TIMEOUT_S overrides.
    double sec = 600.0;
    if (const char* v = getenv("KGP_PEER_TIMEOUT_S")) {
      const double t = atof(v);
      if (t > 0) sec = t;
    }
    e->ptimeout_ns = (unsigned long long)(sec * 1e9);
  }
  for (int q = 0; q <= world; ++q) e->prow[q] = row_start[q];
  for (int q = 0; q < world; ++q) e->pbase[q] = static_cast<uint8_t*>(bases[q]);
  bump_graph_epoch();
  return KGP_OK;
}

// Publish this rank's rows of B for product `epoch` (1, 2, ...): wait until every peer is
// done reading epoch - 1, write the own tiles, then ready = epoch. b_loc must stay valid
// until the matching kgp_engine_peer_matmul (its rows give the + s B term).
extern "C" int kgp_engine_peer_publish(kgp_engine* e, int64_t k, const double* b_loc, int64_t b_rs, int64_t b_cs,
                                       uint64_t epoch, void* stream) {
  CHECK_ENGINE(e);
  int prc = peer_check(e);
  if (prc) return prc;
  KGP_REQUIRE(epoch >= 1 && k >= 1 && b_loc != nullptr, KGP_ERR_INVALID, "bad publish arguments");
  KGP_REQUIRE((k + 15) / 16 <= (e->pkcap + 15) / 16, KGP_ERR_INVALID,
              "RHS block of %lld columns exceeds the peer buffers' capacity (%lld)", (long long)k,
              (long long)e->pkcap);
  const int split = tc_split_of(e->precision);
  KGP_REQUIRE(k <= tc_max_kp(e->dpad, 2, split, 1), KGP_ERR_INVALID,
              "the fused all-gather operator takes one launch's RHS block (k = %lld too wide)", (long long)k);
  KGP_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned long long* f[KGP_MAX_PEERS] = {};
  for (int q = 0; q < e->pworld; ++q) f[q] = reinterpret_cast<const unsigned long long*>(e->pbase[q] + 8);  // done
  peer_wait_done_kernel<<<1, 32, 0, st>>>(e->pworld, e->prank, (unsigned long long)(epoch - 1), e->ptimeout_ns,
                                          f[0], f[1],
                                          f[2], f[3], f[4], f[5], f[6], f[7]);
  KGP_LAUNCH("peer_wait_done_kernel");
  const int kp = (int)((k + 15) / 16 * 16);
  uint8_t* mine = e->pbase[e->prank];
  int rc = prep_rhs(split, 0, e->nrows, k, 0, kp, b_loc, b_rs, b_cs, mine + PEER_HDR, st);
  if (rc) return rc;
  peer_flag_kernel<<<1, 1, 0, st>>>(reinterpret_cast<unsigned long long*>(mine), (unsigned long long)epoch);
  KGP_LAUNCH("peer_flag_kernel");
  e->pb = b_loc;
  e->pb_rs = b_rs;
  e->pb_cs = b_cs;
  e->pk = k;
  return KGP_OK;
}

// This rank's rows of Khat B (and dKhat/dl B, dKhat/df B) for product `epoch`, reading every
// rank's published tiles as the column sweep reaches them; then done = epoch.
extern "C" int kgp_engine_peer_matmul(kgp_engine* e, int64_t k, uint64_t epoch, double* out_k, double* out_dl,
                                      double* out_df, int64_t o_rs, int64_t o_cs, void* stream) {
  CHECK_ENGINE(e);
  int prc = peer_check(e);
  if (prc) return prc;
  KGP_REQUIRE(e->pb != nullptr && k == e->pk, KGP_ERR_STATE, "kgp_engine_peer_publish(k = %lld) must precede",
              (long long)k);
  KGP_REQUIRE(out_k || out_dl || out_df, KGP_ERR_INVALID, "no output requested");
  KGP_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = engine_prepare(e, st);
  if (rc) return rc;
  rc = tc_matmul(e, e->xrow.as<float>(), e->nrows, 0, k, e->pb, e->pb_rs, e->pb_cs, out_k, out_dl, out_df, o_rs,
                 o_cs, st, false, epoch);
  if (rc) return rc;
  peer_flag_kernel<<<1, 1, 0, st>>>(reinterpret_cast<unsigned long long*>(e->pbase[e->prank] + 8),
                                    (unsigned long long)epoch);
  KGP_LAUNCH("peer_flag_kernel");
  return KGP_OK;
}
