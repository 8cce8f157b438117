// Shared device helpers for libkgp (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdio>
#include <stdint.h>

#include "../../include/kgp.h"

#define KGP_DEV __device__ __forceinline__

namespace kgp {

// ---------------------------------------------------------------- error plumbing
void set_error(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);
void count_launches(int64_t n);
#define KGP_CUDA(call)                                         \
  do {                                                         \
    int _rc = ::kgp::cuda_check((call), #call);                \
    if (_rc != KGP_OK) return _rc;                             \
  } while (0)
#define KGP_LAUNCH(what)                                       \
  do {                                                         \
    ::kgp::count_launches(1);                                  \
    int _rc = ::kgp::cuda_check(cudaGetLastError(), what);     \
    if (_rc != KGP_OK) return _rc;                             \
  } while (0)
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device context: raise it once per
// (kernel, device), tracked in a per-call-site bitmask (devices 0..63), thread-safe.
#define KGP_SMEM_ATTR(kern, bytes)                                                                   \
  do {                                                                                               \
    static std::atomic<uint64_t> _kgp_smem_mask{0};                                                  \
    int _dev = 0;                                                                                    \
    KGP_CUDA(cudaGetDevice(&_dev));                                                                  \
    const uint64_t _bit = 1ull << (_dev & 63);                                                       \
    if (!(_kgp_smem_mask.load(std::memory_order_acquire) & _bit)) {                                  \
      KGP_CUDA(cudaFuncSetAttribute((kern), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes))); \
      _kgp_smem_mask.fetch_or(_bit, std::memory_order_acq_rel);                                      \
    }                                                                                                \
  } while (0)
#define KGP_REQUIRE(cond, code, ...)                           \
  do {                                                         \
    if (!(cond)) {                                             \
      ::kgp::set_error((code), __VA_ARGS__);                   \
      return (code);                                           \
    }                                                          \
  } while (0)

// ---------------------------------------------------------------- kernel constants
enum Kern { GAUSS = 0, MAT32 = 1, MAT52 = 2 };

constexpr double SQRT3 = 1.7320508075688772;
constexpr double SQRT5 = 2.23606797749979;
constexpr double LOG2E = 1.4426950408889634;

// ---------------------------------------------------------------- fp64 entry formulas
// The reference panels (_panels_numba.py:37-131), evaluated from r^2.
template <int KT>
KGP_DEV double kappa64(double r2, double l) {
  if (KT == GAUSS) return exp(-r2 * (1.0 / (2.0 * l * l)));
  double t = (KT == MAT32 ? SQRT3 : SQRT5) / l * sqrt(r2);
  if (KT == MAT32) return (1.0 + t) * exp(-t);
  return (1.0 + t + (5.0 / (3.0 * l * l)) * r2) * exp(-t);
}

template <int KT>
KGP_DEV double dkappa64(double r2, double l) {
  if (KT == GAUSS) return r2 * (1.0 / (l * l * l)) * exp(-r2 * (1.0 / (2.0 * l * l)));
  if (KT == MAT32) return (3.0 / (l * l * l)) * r2 * exp(-(SQRT3 / l) * sqrt(r2));
  double t = (SQRT5 / l) * sqrt(r2);
  return (5.0 / (3.0 * l * l * l)) * r2 * (1.0 + t) * exp(-t);
}

// exp(x) for x <= 0 on the FP64 pipe with a short dependency chain, for the fused fp64
// operator whose per-entry cost is the exponential's latency (ncu: stall_wait dominant):
// Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2, exp(r) by its degree-12 Taylor
// polynomial in Estrin form (depth 6 instead of Horner's 12; truncation 1.6e-16 relative),
// 2^k by adding k to the exponent field. A few ulp from the correctly rounded value, against
// the 1e-12 operator bar; results below 2^-1021 (x < -708) are returned as 0. The materialised
// panels keep the library exp (their goldens are compared at 1e-13 entrywise).
KGP_DEV double exp_neg64(double x) {
  if (x < -708.0) return 0.0;
  // k = round(x / ln 2) by the 1.5 * 2^52 shifter: k sits in the low word, no F2I conversion
  const double t = fma(x, LOG2E, 6755399441055744.0);
  const int k = __double2loint(t);
  const double kd = t - 6755399441055744.0;
  const double r = fma(kd, -1.90821492927058770002e-10, fma(kd, -6.93147180369123816490e-01, x));
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  const double p01 = fma(r, 1.0, 1.0);
  const double p23 = fma(r, 1.0 / 6.0, 0.5);
  const double p45 = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  const double p67 = fma(r, 1.0 / 5040.0, 1.0 / 720.0);
  const double p89 = fma(r, 1.0 / 362880.0, 1.0 / 40320.0);
  const double pab = fma(r, 1.0 / 39916800.0, 1.0 / 3628800.0);
  const double q0 = fma(r2, p23, p01);
  const double q1 = fma(r2, p67, p45);
  const double q2 = fma(r4, 1.0 / 479001600.0, fma(r2, pab, p89));
  const double pv = fma(r8, q2, fma(r4, q1, q0));
  return __hiloint2double(__double2hiint(pv) + (k << 20), __double2loint(pv));
}

// Table-driven exp(x) for x <= 0: x = (64 e + j) ln2/64 + r, |r| <= ln2/128, exp(x) =
// 2^e * 2^(j/64) * exp(r) with 2^(j/64) from a 64-entry table in shared memory (`tab`, filled by
// exp_tab_fill) and exp(r) - 1 by its degree-5 Taylor polynomial (truncation r^6/720 <= 3.5e-17):
// 11 FP64 instructions and one LDS against the 19 of exp_neg64 -- the fused fp64 operators are
// bound by the FP64 pipe, the integer/LSU work rides along. The table entries are correctly
// rounded (0.5 ulp), the result is within ~1.5 ulp; x < -708 is clamped to -708 (3.3e-308).
__device__ const double EXP_TAB64[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};

// every thread of the CTA calls this before the first exp_neg64t (the caller synchronises)
KGP_DEV void exp_tab_fill(double* tab) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x) tab[i] = EXP_TAB64[i];
}

KGP_DEV double exp_neg64t(double x, const double* __restrict__ tab) {
  // branch-free: an early return would end the basic block, and the callers rely on the scheduler
  // interleaving this chain with their independent FMA streams. Arguments below -708 evaluate as
  // exp(-708) = 3.3e-308 (instead of a subnormal or 0): an absolute error of 3e-308
  x = fmax(x, -708.0);
  // m = round(64 x / ln 2) by the 1.5 * 2^52 shifter (m in the low word), m = 64 e + j
  const double t = fma(x, 0x1.71547652b82fep+6, 6755399441055744.0);
  const int m = __double2loint(t);
  const double md = t - 6755399441055744.0;
  // r = x - m ln2/64, ln2/64 split so that m * hi is exact (|m| < 2^17, hi has 33 bits)
  const double r = fma(md, -0x1.a39ef35793c76p-39, fma(md, -0x1.62e42fee00000p-7, x));
  const double tj = tab[m & 63];
  const double r2 = r * r;
  const double a = fma(r, 1.0 / 6.0, 0.5);
  const double b = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  const double c = fma(r2, b, a);
  const double q = fma(r2, c, r);       // exp(r) - 1
  const double pv = fma(tj, q, tj);     // 2^(j/64) exp(r), in [0.99, 2.01)
  return __hiloint2double(__double2hiint(pv) + ((m >> 6) << 20), __double2loint(pv));
}

// (the Gaussian keeps the library exp: measured faster there -- cfg2-shape fp64 step 52 vs
// 63 ms -- while the Matern kernels gain 25 %: 2.75 -> 2.05 ms at n = 16384, k = 33)
// FG: the Gaussian's exponential by the branch-free exp_neg64 as well (the library exp's
// slow-path branch splits every entry's evaluation into its own basic block): measured at the
// cfg2 shape (d = 8, k = 32, two outputs) 94.8 -> 55.9 ms; at d = 3 (configs[0]) the library exp
// is 3 % faster, so the operators select it by dimension
// TAB: the exponential by exp_neg64t (table in shared memory) for every kernel type
#ifndef KGP_F64_TABEXP
#define KGP_F64_TABEXP 1
#endif
template <int KT, bool FG>
KGP_DEV double exp_sel(double x, const double* __restrict__ tab) {
#if KGP_F64_TABEXP
  return exp_neg64t(x, tab);
#else
  if (KT == GAUSS && !FG) return exp(x);
  return exp_neg64(x);
#endif
}

template <int KT, bool FG = false>
KGP_DEV double kappa64f(double r2, double l, const double* __restrict__ tab) {
  if (KT == GAUSS) return exp_sel<KT, FG>(-r2 * (1.0 / (2.0 * l * l)), tab);
  double t = (KT == MAT32 ? SQRT3 : SQRT5) / l * sqrt(r2);
  if (KT == MAT32) return (1.0 + t) * exp_sel<KT, FG>(-t, tab);
  return (1.0 + t + (5.0 / (3.0 * l * l)) * r2) * exp_sel<KT, FG>(-t, tab);
}

// kappa and dkappa/dl of one entry from ONE exponential: the same values, bit for bit, as
// kappa64f / dkappa64f (the same expressions, the exponential's argument rounded the same way)
template <int KT, bool FG = false>
KGP_DEV void kd64f(double r2, double l, double& kv, double& gv, const double* __restrict__ tab) {
  if (KT == GAUSS) {
    const double x = -r2 * (1.0 / (2.0 * l * l));
    const double e = exp_sel<KT, FG>(x, tab);
    kv = e;
    gv = r2 * (1.0 / (l * l * l)) * e;
    return;
  }
  const double t = (KT == MAT32 ? SQRT3 : SQRT5) / l * sqrt(r2);
  const double e = exp_sel<KT, FG>(-t, tab);
  if (KT == MAT32) {
    kv = (1.0 + t) * e;
    gv = (3.0 / (l * l * l)) * r2 * e;
  } else {
    kv = (1.0 + t + (5.0 / (3.0 * l * l)) * r2) * e;
    gv = (5.0 / (3.0 * l * l * l)) * r2 * (1.0 + t) * e;
  }
}

template <int KT>
KGP_DEV double dkappa64f(double r2, double l) {
  if (KT == GAUSS) return r2 * (1.0 / (l * l * l)) * exp(-r2 * (1.0 / (2.0 * l * l)));
  if (KT == MAT32) return (3.0 / (l * l * l)) * r2 * exp_neg64(-(SQRT3 / l) * sqrt(r2));
  double t = (SQRT5 / l) * sqrt(r2);
  return (5.0 / (3.0 * l * l * l)) * r2 * (1.0 + t) * exp_neg64(-t);
}

// ---------------------------------------------------------------- warp helpers
KGP_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- PTX: mbarrier / bulk copy / tcgen05
KGP_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

KGP_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
KGP_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
KGP_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
KGP_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
#ifdef KGP_MBAR_DEBUG
KGP_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  for (long long it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (it == (1ll << 24)) {
      printf("mbar hang: block (%d,%d) warp %d lane %d bar+%u parity %u\n", blockIdx.x, blockIdx.y,
             threadIdx.x >> 5, threadIdx.x & 31, addr & 0x3ff, parity);
      __trap();
    }
  }
}
#else
#ifndef KGP_MBAR_HINT
#define KGP_MBAR_HINT 0  // try_wait suspend-time hint (ns); 0: the hardware default window
#endif
KGP_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
#if KGP_MBAR_HINT > 0
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity), "n"(KGP_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
#endif
}
#endif
// mbarrier wait that backs off with __nanosleep between probes: every try_wait is an MIO
// operation, and warps that spin on a barrier for hundreds of cycles (the drain, the producer,
// compute sets waiting for their next stage) throttle the MIO queue that the tcgen05.mma
// issuer and the TMEM loads/stores share. ns = 0: plain spin.
KGP_DEV bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
KGP_DEV void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns) {
  if (ns == 0) {
    mbar_wait(bar, parity);
    return;
  }
  while (!mbar_try(bar, parity)) __nanosleep(ns);
}

// 1-D bulk async copy global -> shared, completion signalled on an mbarrier (tx bytes).
KGP_DEV void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- cross-GPU flags (fused all-gather)
// Bounded wait for a peer's flag (system-scope acquire): a peer that never arrives traps the
// kernel after `timeout_ns` instead of hanging the device. A trap is a sticky CUDA error:
// the process's context is lost, so the bound (KGP_PEER_TIMEOUT_S, default 600 s) must sit
// far above any host-side skew between ranks; dist.py barriers at set_peers and before the
// first publish so only device progress is ever waited on.
KGP_DEV void peer_wait_flag(const unsigned long long* flag, unsigned long long want,
                            unsigned long long timeout_ns) {
  unsigned long long t0, now, v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= want) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > timeout_ns) {
      printf("kgp: peer flag %p stuck at %llu (want %llu)\n", (const void*)flag, v, want);
      __trap();
    }
    __nanosleep(128);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");  // later bulk copies read what the flag released
}
KGP_DEV void peer_set_flag(unsigned long long* flag, unsigned long long v) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
}

// One lane of a converged warp (elect.sync): the single issuing thread for
// tcgen05.mma / bulk copies, without a divergent `lane == 0` region that would
// force the compiler to waterfall the (warp-uniform) operands into uniform registers.
KGP_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
      "elect.sync rx|px, %1;\n\t"
      "@px mov.s32 %0, 1;\n\t}"
      : "+r"(pred)
      : "r"(0xFFFFFFFFu));
  return pred != 0;
}

KGP_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
KGP_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
KGP_DEV void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
KGP_DEV void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// wait::ld that also "redefines" the destination registers of an earlier asynchronous
// tcgen05.ld, so the compiler cannot hoist their uses above the wait
KGP_DEV void tc_wait_ld_tied(uint32_t (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}

// Commit all prior tcgen05.mma of this thread to an mbarrier (one arrival when they finish).
KGP_DEV void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem desc], kind::tf32, cta_group::1.
KGP_DEV void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem desc], kind::f16 (bf16 inputs per idesc), cta_group::1.
// A in TMEM packs two 16-bit K elements per 32-bit column (lower K index in the low half).
KGP_DEV void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

// 32 lanes x 32 bit, 8 consecutive columns.
KGP_DEV void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns: thread t <-> lane (quadrant base + t).
KGP_DEV void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// 16 lanes x 256 bit, twice along columns (16 columns): thread t holds lanes {t/4, t/4+8}
// (relative to the address lane) and columns {2(t%4), 2(t%4)+1} (+8 for the second half):
// v[0..1] = (t/4, c..c+1), v[2..3] = (t/4+8, c..c+1), v[4..5] = (t/4, c+8..c+9), v[6..7] = (t/4+8, c+8..c+9).
KGP_DEV void tmem_st_16x256b_x2(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
// .x4: four 8-column groups (32 columns); group m occupies v[4m .. 4m+3] in the .x2 order
KGP_DEV void tmem_st_16x256b_x4(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
KGP_DEV void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
KGP_DEV void tmem_ld_16x256b_x2(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc], kind::tf32, cta_group::1.
KGP_DEV void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
// Make generic-proxy shared-memory writes visible to the async proxy (tensor core reads).
KGP_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
KGP_DEV void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15])
      : "r"(taddr)
      : "memory");
}


// 32 lanes x 32 bit, 32 consecutive columns (one instruction: half the MIO operations of two x16)
KGP_DEV void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr)
               : "memory");
}
KGP_DEV void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
               : "memory");
}
KGP_DEV void tc_wait_ld_tied32(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31]) : : "memory");
}

template <int NCOLS>
KGP_DEV void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
KGP_DEV void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B apart.
// Fields (sm100): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version=1 [46,48),
// base offset [49,52), layout type [61,64) (2 = SWIZZLE_128B).
KGP_DEV uint64_t sw128_kmajor_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;            // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

// UMMA shared-memory descriptor: K-major, no swizzle ("interleaved"): core matrices of
// 8 rows x 16 B stored contiguously (128 B); `lbo` = byte distance between the two
// 16-byte K chunks of one MMA, `sbo` = byte distance between 8-row groups.
KGP_DEV uint64_t interleave_kmajor_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell); layout type 0 = SWIZZLE_NONE
  return d;
}

// Byte offset of element (row r, k) in a K-major no-swizzle tf32 tile with `rows` rows.
// Tensor-core distance operands (d > 4): U'_i = [-2 gamma c_i (dpad) | q_i hi, q_i lo, 1, 1 | 0..]
// and V'_j = [c_j (dpad) | 1, 1, q_j hi, q_j lo | 0..], q = gamma |c|^2 split into an exact tf32
// head and its remainder. t2 = U'.V' then needs the tf32 lo parts of the coordinates only, so
// the 3xTF32 product is hi.hi over all K plus hi.lo and lo.hi over the first dpad columns: 4
// MMAs per block at dpad = 8 instead of 6 with [u, q, 1] . [c, 1, q] (KGP_TC_DIST4 0)
#ifndef KGP_TC_DIST4
#define KGP_TC_DIST4 1
#endif
__host__ __device__ constexpr int tc_dist_kd(int dpad) { return ((dpad + (KGP_TC_DIST4 ? 4 : 2)) + 7) / 8 * 8; }

__host__ __device__ inline uint32_t interleave_offset(uint32_t r, uint32_t k, uint32_t rows) {
  return (k >> 2) * (rows * 16u) + (r >> 3) * 128u + (r & 7u) * 16u + (k & 3u) * 4u;
}

// Instruction descriptor, kind::tf32: D=F32, A=B=TF32, both K-major, M=128, N=n.
__host__ __device__ constexpr uint32_t idesc_tf32_m128(int n) {
  return (1u << 4)                       // D format F32
         | (2u << 7)                     // A format TF32
         | (2u << 10)                    // B format TF32
         | ((uint32_t)(n >> 3) << 17)    // N >> 3
         | ((uint32_t)(128 >> 4) << 24); // M >> 4
}

// Instruction descriptor, kind::f16: D=F32, A=B=BF16, both K-major, M=128, N=n.
__host__ __device__ constexpr uint32_t idesc_bf16_m128(int n) {
  return (1u << 4)                       // D format F32
         | (1u << 7)                     // A format BF16
         | (1u << 10)                    // B format BF16
         | ((uint32_t)(n >> 3) << 17)    // N >> 3
         | ((uint32_t)(128 >> 4) << 24); // M >> 4
}

// Byte offset of element (row r, k) in a K-major no-swizzle 16-bit tile with `rows` rows
// (core matrices of 8 rows x 8 elements, K chunks `rows` x 16 B apart).
__host__ __device__ inline uint32_t interleave16_offset(uint32_t r, uint32_t k, uint32_t rows) {
  return (k >> 3) * (rows * 16u) + (r >> 3) * 128u + (r & 7u) * 16u + (k & 7u) * 2u;
}

// Byte offset of element (row r, k-index j) of a K-major fp32 tile whose rows are
// 128 B (32 elements), under the 128-byte swizzle (Swizzle<3,4,3>).
__host__ __device__ inline uint32_t sw128_offset(uint32_t r, uint32_t j) {
  uint32_t o = r * 128u + j * 4u;
  return o ^ (((o >> 7) & 7u) << 4);
}

}  // namespace kgp
