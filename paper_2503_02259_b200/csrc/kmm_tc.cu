// Fused kernel-matrix MatMul on the 5th-generation tensor cores (sm_100a).
//
// Replaces KernelEngine._streamed_matmul (kmat.py:165-189) and the numba panels
// (_panels_numba.py:37-131) for precision KGP_FAST / KGP_TF32:
//
//   acc_K = kappa(X_rows, X) . B        acc_G = (scaled dkappa/dl)(X_rows, X) . B
//
// The kernel matrix is never stored. One CTA owns 128 rows (the TMEM lanes) and
// streams the columns in blocks of 32 (one 128-byte swizzle atom of tf32). With NS
// compute-warp sets (2 or 3, ns_for) the warps are:
//   * compute (4*NS warps, one per TMEM lane quadrant per set; set e takes the blocks
//     t = e mod NS): read the block's squared distances, apply the kernel transform (MUFU
//     ex2/sqrt), split into tf32 hi/lo and store the tile into TMEM with tcgen05.st -- the
//     A operand of the contraction (16x256b layout, or 32x32b for the fused two-output
//     3xTF32 product);
//   * producer (1): cp.async.bulk of each block's operands into a 4/8-stage SMEM ring: the
//     RHS tiles, pre-split into tf32 hi/lo and already in the UMMA K-major 128B-swizzled
//     layout, plus the block's column-point data;
//   * contraction MMA issuer (1): tcgen05.mma kind::tf32, cta_group::1, A from TMEM, B from
//     SMEM, one elected lane of a converged warp: hi*hi + hi*lo + lo*hi per output and K=8
//     chunk (3xTF32; hi*hi only for KGP_TF32);
//   * distance MMA issuer (1, d > 4): the scaled squared distance t2 = gamma r^2 is itself
//     an MMA: with U'_i = [-2 gamma c_i, q_i, 1] (resident in TMEM) and V'_j = [c_j, 1, q_j]
//     (q = gamma |c|^2, c centred), t2 = U' V'^T, a K = d+2 (padded to 16) 3xTF32 product
//     into a per-set TMEM buffer, issued as soon as a block's V' lands. (d <= 4 keeps
//     direct differences on the FP32 pipe in the compute warps: cheaper there and exact for
//     near-coincident points);
//   * drain (4): every `flush` blocks promote the TMEM accumulators into fp32 shared-memory
//     sums (two buffers ping-pong, or one when the RHS block is wide). The tensor core's
//     fp32 accumulation truncates: unpromoted it drifts linearly in n (measured 4.6e-4 at
//     n = 65536); promoted it stays near 2e-6.
// The drain warps finally apply f^2, 2f, s*B and the derivative scale in fp64 (or write
// fp32 partials when the column sweep is split over grid.y; tc_reduce_kernel finishes).
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdlib.h>

#include "kgp_common.cuh"
#include "kgp_internal.h"

namespace kgp {

namespace {

#ifndef KGP_TC_RACC
#define KGP_TC_RACC 1  // drain: promotion sums in registers when the RHS block has <= 64 columns
#endif
// Backoff (ns) of the mbarrier waits by role (0 = spin): see mbar_wait_backoff
#ifndef KGP_TC_SLEEP_DRAIN
#define KGP_TC_SLEEP_DRAIN 0
#endif
#ifndef KGP_TC_SLEEP_COMP
#define KGP_TC_SLEEP_COMP 0
#endif
#ifndef KGP_TC_SLEEP_PROD
#define KGP_TC_SLEEP_PROD 0
#endif

// Compute warp sets: set e handles blocks t = e (mod NS); every ring a set touches (TMEM
// A stages, distance buffers) has NS slots so each slot has exactly one writer set.
// NS = 2 when the A stages are wide (two outputs, hi/lo), 3 otherwise (TMEM budget).
#ifndef KGP_TC_NSET
#define KGP_TC_NSET 0  // 0: per-configuration default (ns_for)
#endif
#ifndef KGP_TC_BF_NS
#define KGP_TC_BF_NS 3  // compute sets of the bf16x3 kernels
#endif
constexpr int ns_for(int nout, int split) {
  return KGP_TC_NSET ? KGP_TC_NSET : (split == 2 ? KGP_TC_BF_NS : ((nout == 2 && split == 3) ? 2 : 3));
}
constexpr int WPS = 4;                    // warps per set = one per TMEM lane quadrant
constexpr int MAXNS = 4;
constexpr int MAXNSB = 8;                 // shared-memory ring depth: runtime p.nsb in {4, 8}
constexpr int BJ = 32;                    // columns per block
constexpr int nthreads_for(int ns) { return (ns * WPS + 7) * 32; }  // + producer, 2 MMA issuers, 4 drain
// LB layouts (below): 1 = two compute sets and three A stages, 2 = three sets and three stages
constexpr int ns_of(int nout, int split, int lbm) { return lbm == 2 ? 3 : ns_for(nout, split); }

KGP_DEV float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
KGP_DEV float sqrtf_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#ifndef KGP_TC_SQRT_FMA
#define KGP_TC_SQRT_FMA 0  // measured: Matern-3/2 d=4 k=33 one output 2.95 -> 4.19 ms (issue-bound, not XU-bound)
#endif
KGP_DEV float2 hi2(float2 v) {
  return make_float2(__uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
}
KGP_DEV float2 fsub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
KGP_DEV float2 lo2(float2 v) { return fsub2(v, hi2(v)); }

#ifndef KGP_TC_DMIN
#define KGP_TC_DMIN 4  // padded dimensions <= DMIN use direct differences, larger the tensor-core distance
#endif
#ifndef KGP_TC_XP
#define KGP_TC_XP 0  // measured: the FP32 expansion is slower than the tensor-core distance at d = 8 (FP32-pipe bound)
#endif

// 2^x (x <= 0) on the FMA pipe instead of MUFU: x = n + f (n = rint(x) by the 1.5 * 2^23 shift,
// |f| <= 1/2), degree-5 minimax p(f) (relative error 2.3e-7 with fp32 Horner, the same class as
// ex2.approx's), exponent field += n by one LEA. x is clamped at -125 (2^-125 is zero next to
// the tile's 1e-7 relative error; ex2.approx.ftz flushes there). MUFU ops go through the SM's
// MIO queue, which the tcgen05.mma issue shares: moving some of the
// exponentials onto the FMA pipe shortens that queue.
#ifndef KGP_TC_LEAN
#define KGP_TC_LEAN 1  // MMA warp skips the full[s] wait, distance warp skips its empty[s] commit
#endif
#ifndef KGP_TC_LRX
#define KGP_TC_LRX 1  // lean form for the direct-difference kernels where it measured faster (LRX)
#endif
#ifndef KGP_TC_PRE
#define KGP_TC_PRE 0  // 16-column halves transformed before the A-stage wait (fused 32x32b path)
#endif
#ifndef KGP_TC_EXPPOLY
#define KGP_TC_EXPPOLY 0  // column pairs (of 8 per 16-column half) whose exp2 runs on the FMA pipe
#endif
KGP_DEV float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 y = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
  const float2 n = __fadd2_rn(y, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = fsub2(x, n);
  float2 p = __ffma2_rn(f, make_float2(0.0013276470126584172f, 0.0013276470126584172f),
                        make_float2(0.009675540961325169f, 0.009675540961325169f));
  p = __ffma2_rn(f, p, make_float2(0.05550713464617729f, 0.05550713464617729f));
  p = __ffma2_rn(f, p, make_float2(0.24022120237350464f, 0.24022120237350464f));
  p = __ffma2_rn(f, p, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = __ffma2_rn(f, p, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(y.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(y.y) << 23)));
}

// Kernel transform of the scaled squared distance t2 = gamma r^2 (see prep.cu):
//   Gaussian  t2 = r^2 log2(e) / (2 l^2)   kappa = 2^-t2              g = t2 kappa
//   Matern32  t2 = 3 r^2 / l^2             kappa = (1+t) e^-t         g = t2 e^-t
//   Matern52  t2 = 5 r^2 / l^2             kappa = (1+t+t2/3) e^-t    g = t2 (1+t) e^-t
// with t = sqrt(t2); dkappa/dl = scale_dl * g (scale folded into the epilogue).
// CLAMP: t2 from the expansion can cancel below zero (_panels_numpy.py:26-27); direct
// differences (d <= 4) are a sum of squares and skip the clamp (one FMNMX per entry).
// The clamp costs one FMNMX per entry in issue-bound compute warps, so it is not an
// instruction: the Gaussian takes t2 as is (a cancelled t2 = -eps gives kappa = 1 + eps ln 2 and
// g = -eps, both within the fp32 tile's own error of the clamped values), and the Matern
// square root reads |t2| (a free source modifier); only the XP (FP32-expansion) path, which
// can cancel further, keeps FMNMX.
template <int KT, bool NEED_G, bool CLAMP = true, bool POLY = false>
KGP_DEV void transform2(float2 t2, float2& kv, float2& gv) {
  if (CLAMP && KGP_TC_XP) {
    t2.x = fmaxf(t2.x, 0.0f);
    t2.y = fmaxf(t2.y, 0.0f);
  }
  if (KT == GAUSS) {
    kv = POLY ? ex2_poly2(make_float2(-t2.x, -t2.y)) : make_float2(ex2f(-t2.x), ex2f(-t2.y));
    if (NEED_G) gv = __fmul2_rn(t2, kv);
  } else {
#if KGP_TC_SQRT_FMA
    // sqrt on the FMA pipe (the MUFU/XU pipe is the busiest one for Matern): rsqrt seed by the
    // exponent-halving bit trick, three Newton steps, t = t2 * rsqrt(t2)
    const float2 hx = __fmul2_rn(t2, make_float2(0.5f, 0.5f));
    float2 y = make_float2(__uint_as_float(0x5f375a86u - (__float_as_uint(t2.x) >> 1)),
                           __uint_as_float(0x5f375a86u - (__float_as_uint(t2.y) >> 1)));
#pragma unroll
    for (int it = 0; it < 3; ++it) {
      const float2 h = __fmul2_rn(hx, y);
      const float2 e = __ffma2_rn(make_float2(-h.x, -h.y), y, make_float2(1.5f, 1.5f));
      y = __fmul2_rn(y, e);
    }
    float2 t = __fmul2_rn(t2, y);  // t2 = 0: y is finite (seed of +0), t = 0
#else
    float2 t = make_float2(sqrtf_approx(fabsf(t2.x)), sqrtf_approx(fabsf(t2.y)));
#endif
    float2 a = __fmul2_rn(t, make_float2(-1.4426950408889634f, -1.4426950408889634f));
    float2 e = make_float2(ex2f(a.x), ex2f(a.y));
    float2 u = __ffma2_rn(t, e, e);  // (1+t) e^-t
    if (KT == MAT32) {
      kv = u;
      if (NEED_G) gv = __fmul2_rn(t2, e);
    } else {
      kv = __ffma2_rn(__fmul2_rn(t2, make_float2(1.0f / 3.0f, 1.0f / 3.0f)), e, u);
      if (NEED_G) gv = __fmul2_rn(t2, u);
    }
  }
}

// register order of tcgen05 16x256b.x4 for one thread: for column group m (columns
// c + 8m, c = 2(t%4)): (row r: 2 regs), (row r+8: 2 regs)
KGP_DEV void pack16(uint32_t (&w)[16], const float2 (&v)[2][4], int mode) {
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    float2 a = v[0][m], b = v[1][m];
    if (mode == 1) { a = hi2(a); b = hi2(b); }
    if (mode == 2) { a = lo2(a); b = lo2(b); }
    w[4 * m] = __float_as_uint(a.x); w[4 * m + 1] = __float_as_uint(a.y);
    w[4 * m + 2] = __float_as_uint(b.x); w[4 * m + 3] = __float_as_uint(b.y);
  }
}

template <int SPLIT>
KGP_DEV void store_tile(uint32_t taddr, const float2 (&v)[2][4]) {
  uint32_t w[16];
  if (SPLIT == 3) {
    pack16(w, v, 1);
    tmem_st_16x256b_x4(taddr, w);
    pack16(w, v, 2);
    tmem_st_16x256b_x4(taddr + 32, w);
  } else {
    pack16(w, v, 0);
    tmem_st_16x256b_x4(taddr, w);
  }
}

// 32x32b layout (thread = one TMEM lane/row, registers = 16 consecutive columns)
#ifndef KGP_TC_ST8
#define KGP_TC_ST8 1  // x8 tcgen05.st (4: x4, 0: x16): cfg2 x16 3.286, x8 3.246, x4 3.300 ms; tools/tc_probe.py
#endif
KGP_DEV void st16_maybe_split(uint32_t taddr, const uint32_t (&w)[16]) {
#if KGP_TC_ST8 == 4
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr + 4 * q),
                 "r"(w[4 * q]), "r"(w[4 * q + 1]), "r"(w[4 * q + 2]), "r"(w[4 * q + 3])
                 : "memory");
#elif KGP_TC_ST8
  uint32_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = w[i];
    b[i] = w[8 + i];
  }
  tmem_st8(taddr, a);
  tmem_st8(taddr + 8, b);
#else
  tmem_st16(taddr, w);
#endif
}
template <int SPLIT>
KGP_DEV void store_row16(uint32_t taddr, const float2 (&v)[8]) {
  uint32_t w[16];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const float2 h = SPLIT == 3 ? hi2(v[m]) : v[m];
    w[2 * m] = __float_as_uint(h.x);
    w[2 * m + 1] = __float_as_uint(h.y);
  }
  st16_maybe_split(taddr, w);
  if (SPLIT == 3) {
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float2 l = lo2(v[m]);
      w[2 * m] = __float_as_uint(l.x);
      w[2 * m + 1] = __float_as_uint(l.y);
    }
    st16_maybe_split(taddr + 32, w);
  }
}

// bf16x3 layout: 16 columns of one row as two round-to-nearest bf16 terms A0 + A1 (8 bf16
// pairs each, lower K in the low half): A0 at a0addr, A1 at a1addr (8 TMEM columns each)
KGP_DEV void store_row16_bf(uint32_t a0addr, uint32_t a1addr, const float2 (&v)[8]) {
  uint32_t w0[8], w1[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const __nv_bfloat162 b0 = __floats2bfloat162_rn(v[m].x, v[m].y);
    const float2 f0 = __bfloat1622float2(b0);
    const float2 r = fsub2(v[m], f0);
    const __nv_bfloat162 b1 = __floats2bfloat162_rn(r.x, r.y);
    w0[m] = *reinterpret_cast<const uint32_t*>(&b0);
    w1[m] = *reinterpret_cast<const uint32_t*>(&b1);
  }
  tmem_st8(a0addr, w0);
  tmem_st8(a1addr, w1);
}

// LB layout: 16 columns of one row as tf32 hi (truncated, 16 TMEM columns at taddr)
// and the lo parts as 8 bf16 pairs (8 columns at the output's lo base + 8 per half)
KGP_DEV void store_row16_lb(uint32_t taddr, uint32_t laddr, const float2 (&v)[8]) {
  uint32_t w[16], wl[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const float2 h = hi2(v[m]);  // truncation: one LOP per value (cvt.rna costs four)
    w[2 * m] = __float_as_uint(h.x);
    w[2 * m + 1] = __float_as_uint(h.y);
    const float2 lo = fsub2(v[m], h);
    const __nv_bfloat162 b = __floats2bfloat162_rn(lo.x, lo.y);  // .x (lower K) in the low half
    wl[m] = *reinterpret_cast<const uint32_t*>(&b);
  }
  tmem_st16(taddr, w);
  tmem_st8(laddr, wl);
}

// Compute-warp TMEM layout: 32x32b (thread = row, 16 columns per op) or 16x256b (thread =
// 4 rows x 8 columns). Measured at cfg2 shape: 32x32b is 8.5% faster for the fused
// two-output 3xTF32 product, 16x256b 1-2% faster for the others (and clearly faster for
// the direct-difference d <= 4 path, whose 4x8 register tile reuses the column data).
#ifndef KGP_TC_LD32
#define KGP_TC_LD32 1
#endif
constexpr bool use_ld32(int nout, int split, bool dmma) {
  return dmma && ((KGP_TC_LD32 && nout == 2 && split == 3) || split == 2);  // bf16x3: row layout only
}

template <int D>
struct Geo {
  // d > 4: t2 by the expansion q_i + q_j + u_i.v_j, on the FP32 pipe (XP) or as a tensor-core
  // MMA into TMEM (DMMA); d <= 4: direct differences on the FP32 pipe
  static constexpr bool XP = (D > KGP_TC_DMIN) && KGP_TC_XP;
  static constexpr bool DMMA = (D > KGP_TC_DMIN) && !KGP_TC_XP;
  static constexpr int KD = tc_dist_kd(D);                   // augmented K of the distance MMA
  static constexpr uint32_t VBYTES = DMMA ? 2u * BJ * KD * 4u : (uint32_t)(D + 1) * BJ * 4u;  // per block
  static constexpr uint32_t UBYTES = 0u;  // U' lives in TMEM
};

// LB layout (fused two-output 3xTF32, tensor-core distance): each output's A tile is its tf32
// hi part (32 TMEM columns) plus its lo part packed as bf16 pairs (16 columns); the
// corrections are hi*B_lo (tf32) and lo*bf16(B) (kind::f16, K=16), so an A stage takes 96
// columns instead of 128 and TMEM holds three of them. Error terms: |lo| < 2^-10 |A|
// (truncated hi), bf16 rounding 2^-9 of lo and of B -> 2^-18 |A||B| per product.
// Pipeline trace (diagnostic, env KGP_TC_TRACE): clock64 of event `ev` for block `t` in CTA (0, 0).
#ifndef KGP_TC_INSTR
#define KGP_TC_INSTR 0  // 1: compile the pipeline trace and the store/load-skipping diagnostics
#endif
#define KGP_TR(ev, t)                                                                                       \
  do {                                                                                                      \
    if (KGP_TC_INSTR && p.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && (t) < 256 && (threadIdx.x & 31) == 0) { \
      unsigned long long _c;                                                                                \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(_c));                                                    \
      p.trace[(ev) * 256 + (t)] = _c;                                                                       \
    }                                                                                                       \
  } while (0)

template <int KT, int D, int NOUT, int SPLIT, int LBM>
__global__ void __launch_bounds__(nthreads_for(ns_of(NOUT, SPLIT, LBM)), 1) kmm_tc_kernel(const TcParams p) {
  constexpr bool LB = (LBM == 1 || LBM == 2);
  // W2 (LBM 3, fused two-output 3xTF32, kp <= 32): hi*[B_hi | B_lo] as ONE N = 2kp MMA and lo*B_hi
  // as an N = kp MMA into the first half of the same accumulator: 16 contraction MMAs per block
  // instead of 24, the same tensor-pipe time (N = 64 runs at ~2x the N = 32 cycles), fewer issue
  // slots for the MMA warp (the kernel's bottleneck). Accumulator per output:
  // [hi B_hi + lo B_hi | hi B_lo] (2kp columns, one buffer), summed pairwise by the drain.
  constexpr bool W2 = LBM == 3;
  static_assert(!W2 || (NOUT == 2 && SPLIT == 3), "W2 layout: fused two-output 3xTF32");
  constexpr int NS = ns_of(NOUT, SPLIT, LBM);
  // sets, distance buffers, A stages. LBM 1: a third A stage written alternately by the two
  // sets (a stage is rewritten only after the MMAs of the block three back have read it, so
  // a parity wait is never two phases behind); LBM 2: three sets, one per A stage, and two
  // distance buffers the sets take in turn. "Distance ready" is signalled per SET (dfull[set],
  // one completion per block of that set), never per buffer: with three sets on two buffers a
  // buffer's parity could not tell a set's block from the one two turns earlier
  constexpr int NSET = NS, ND = (LBM == 2) ? 2 : NS, NSA = LB ? 3 : NS;
  constexpr int NCW = NS * WPS;                 // compute warps
  constexpr int WPROD = NCW, WMMA = NCW + 1, WDIST = NCW + 2;
  static_assert(NS <= MAXNS, "ring slots");
  using G = Geo<D>;
  constexpr bool DMMA = G::DMMA;
  constexpr bool XP = G::XP;
  constexpr int KD = G::KD;
  constexpr int KDS = (KD + 15) / 16 * 16;  // TMEM column stride of U' hi -> lo
  constexpr int TPO = (SPLIT == 3) ? 2 : 1;  // TMEM tiles per output (hi, lo)
  constexpr int ATILES = NOUT * TPO;
  constexpr int OCOLS = LB ? 48 : TPO * 32;         // TMEM columns per output in an A stage
  constexpr int ASTAGE = NOUT * OCOLS;
  static_assert(!LB || (NOUT == 2 && SPLIT == 3), "LB layout: fused two-output 3xTF32");
  constexpr uint32_t VBYTES = G::VBYTES;
  constexpr bool NEED_G = (NOUT == 2);
  // Runtime diagnostic switches (KGP_TC_DEBUG) in the MMA loop and the 16x256b transform: the
  // tensor-core-distance kernels compile them out (cfg2 3.33 -> 3.15 ms: the dead branches cost
  // the compute and MMA warps issue slots and predicated copies); of the direct-difference
  // kernels only the LRX ones do (Matern-3/2 d=4 k=33 one output: 2.83 ms with them, 3.05
  // without; tools/gpu_ab.sh)
  // LRX: the direct-difference kernels that measured faster with the lean variants too
  // (compiled-out switches, no full-stage wait in the MMA warp; tools/gpu_direct2.sh, n = 65536):
  // two outputs (k = 1-33: 10-20 % faster, k = 64: 2-5 % slower), d <= 2 and the Gaussian (k >= 33:
  // 7-10 % faster, k <= 16: within 3 %). Matern with d = 3..4 and one output (the configs[2]
  // PCG product) measured up to 20 % slower lean and keeps the original form
  constexpr bool LRX = KGP_TC_LRX && (NOUT == 2 || D <= 2 || KT == GAUSS);
  constexpr bool RTD = (!Geo<D>::DMMA && !LRX) || KGP_TC_INSTR;
  if (p.gate != nullptr && *p.gate == 0) return;  // PCG iteration past convergence: nothing to do

  extern __shared__ __align__(1024) uint8_t smem[];
  const int KP = p.kp;
  const int NSB = p.nsb;                           // 4 or 8
  const int nsb_log = (NSB == 8) ? 3 : 2;
  const int NACC = (W2 ? 2 : 1) * NOUT * KP;       // accumulator columns per buffer (TMEM)
  const uint32_t BBYTES = (uint32_t)((TPO * 128 + (LB ? 64 : 0)) * KP);  // tf32 hi | lo (| bf16)
  uint8_t* sB = smem;                              // NSB x BBYTES, 1024-aligned
  uint8_t* sV = smem + NSB * BBYTES;               // NSB x VBYTES (column data / V' tiles)
  uint8_t* sU = sV + NSB * VBYTES;                 // U' hi/lo (DMMA)
  float* sAcc = reinterpret_cast<float*>(sU + G::UBYTES);  // NOUT * KP x 128 fp32, column-major
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAcc + NOUT * KP * 128);
  uint64_t* full = bars;
  uint64_t* empty = bars + MAXNSB;
  uint64_t* afull = bars + 2 * MAXNSB;
  uint64_t* aempty = afull + MAXNS;
  uint64_t* accfull = aempty + MAXNS;
  uint64_t* accempty = accfull + 2;
  uint64_t* dfull = accempty + 2;
  uint64_t* dempty = dfull + MAXNS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + MAXNS);
  static_assert(8 * (2 * MAXNSB + 4 * MAXNS + 4) + 4 <= 512, "barrier area");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int NAB = p.nab;                           // accumulator buffers (2: ping-pong with the drain)
  const int dbase = NAB * NACC;                    // distance buffers follow the accumulators
  const int ucol = dbase + (DMMA ? ND * BJ : 0);   // then U' hi | lo (KD columns each)
  const int abase = ucol + (DMMA ? 2 * KDS : 0);   // then the A stages
  // column split (grid.y): this CTA sweeps column blocks [t0, t0 + nblk)
  const int t0 = p.tbeg + blockIdx.y * p.nper;
  const int nblk = (p.nblk - t0) < p.nper ? (p.nblk - t0) : p.nper;
  const int flush = p.flush;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSB; ++s) {
      mbar_init(&full[s], 1);
      // DMMA: released by the contraction warp's commit alone when KGP_TC_LEAN (the distance MMAs
      // that read the stage's V' completed before dfull, hence before the tile they feed exists)
      mbar_init(&empty[s], DMMA ? (KGP_TC_LEAN ? 1 : 2) : 1 + WPS);
    }
    for (int a = 0; a < NSA; ++a) {
      mbar_init(&afull[a], WPS);
      mbar_init(&aempty[a], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], 4);
    }
    for (int b = 0; b < NSET; ++b) mbar_init(&dfull[b], 1);  // one per compute set
    for (int b = 0; b < ND; ++b) mbar_init(&dempty[b], WPS);  // one per distance buffer
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (DMMA && warp < 4) {
    // U'_r = [-2 gamma c_r (D), q_r, 1, 0 ...] as tf32 hi / lo in TMEM (A operand of the
    // distance MMA): warp w writes lanes 32w..32w+31 (thread = row), KD columns each
    const int r = threadIdx.x;
    const int64_t gr = (int64_t)blockIdx.x * 128 + r;
    const bool ok = gr < p.nrows;
    const float* xr = p.xrow + (ok ? gr : 0) * (D + 1);
    const uint32_t uaddr = tbase + ((uint32_t)(warp * 32) << 16) + ucol;
#pragma unroll
    for (int k0 = 0; k0 < KD; k0 += 16) {
      uint32_t hv[16], lv[16];
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int k = k0 + kk;
        float v = 0.f;
        float hi, lo;
        if (KGP_TC_DIST4) {
          // [u (D) | q hi, q lo, 1, 1]: only the coordinates carry a lo part
          const float q = ok ? xr[0] : 0.0f;
          const float qh = __uint_as_float(__float_as_uint(q) & 0xFFFFE000u);
          if (ok && k < D) v = xr[1 + k];
          else if (ok && k == D) v = qh;
          else if (ok && k == D + 1) v = q - qh;
          else if (ok && (k == D + 2 || k == D + 3)) v = 1.0f;
          hi = (k < D) ? __uint_as_float(__float_as_uint(v) & 0xFFFFE000u) : v;
          lo = (k < D) ? v - hi : 0.0f;
        } else {
          if (ok && k < KD) v = (k < D) ? xr[1 + k] : (k == D ? xr[0] : (k == D + 1 ? 1.0f : 0.0f));
          hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
          lo = v - hi;
        }
        hv[kk] = __float_as_uint(hi);
        lv[kk] = __float_as_uint(lo);
      }
      tmem_st16(uaddr + k0, hv);
      tmem_st16(uaddr + KDS + k0, lv);
    }
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == WPROD) {
    // ------------------------------------------------------------ producer (converged warp, one elected issuer)
    int s = 0, owner = -1;
    uint32_t ph = 0;
    for (int t = 0; t < nblk; ++t) {
      mbar_wait_backoff(&empty[s], ph ^ 1, KGP_TC_SLEEP_PROD);
      KGP_TR(0, t);
      const uint8_t* bsrc = p.bsplit + (size_t)(t0 + t) * BBYTES;
      if (p.npeer > 0) {  // fused all-gather: this block's RHS tile lives in its owner's buffer
        const int tg = t0 + t;
        int q = owner < 0 ? 0 : owner;
        while (q + 1 < p.npeer && tg >= p.pblk0[q + 1]) ++q;
        if (q != owner) {  // first block of this owner in the sweep: wait for its tiles
          if (elect_one()) peer_wait_flag(p.pready[q], p.epoch, p.ptimeout_ns);
          __syncwarp();
          owner = q;
        }
        bsrc = p.ptile[q] + (size_t)(tg - p.pblk0[q]) * BBYTES;
      }
      if (elect_one()) {
        mbar_arrive_expect_tx(&full[s], BBYTES + VBYTES);
        bulk_g2s(sB + s * BBYTES, bsrc, BBYTES, &full[s]);
        bulk_g2s(sV + s * VBYTES, reinterpret_cast<const uint8_t*>(p.xcol) + (size_t)(t0 + t) * VBYTES, VBYTES, &full[s]);
      }
      __syncwarp();
      if (++s == NSB) { s = 0; ph ^= 1; }
    }
  } else if (warp == WMMA) {
    // ------------------------------------------------------------ contraction MMA issuer (converged warp)
    const uint32_t idesc = idesc_tf32_m128(KP);
    int s = 0, a = 0, pos = 0, ab = 0;
    uint32_t ph_s = 0, ph_a = 0, ph_acc = 0;
    for (int t = 0; t < nblk; ++t) {
      if (pos == 0) mbar_wait(&accempty[ab], ph_acc ^ 1);  // buffer drained (segment start)
      // KGP_TC_LEAN: no wait on full[s]. The A tile of block t exists only after its compute set
      // saw the block's distances (DMMA: issued after the distance warp saw full[s]) or its
      // column data (direct path: the set itself waits on full[s]), so afull[a] completing
      // already orders this warp after the stage's bulk copies (acquire chains through the
      // barriers); every mbarrier probe is an MIO round trip on the issuer's critical path.
      // (Measured: cfg2 3.13 -> 3.02 ms; on the direct-difference path, whose sets wait on
      // full[s] themselves, dropping it made Matern-3/2 d=4 slower, so it stays there)
      if (!(KGP_TC_LEAN && (DMMA || LRX))) mbar_wait(&full[s], ph_s);
      mbar_wait(&afull[a], ph_a);
      tc_fence_after();
      KGP_TR(7, t);
      const uint32_t bhi = smem_u32(sB + s * BBYTES);
      const uint64_t dhi = sw128_kmajor_desc(bhi);
      const uint64_t dlo = sw128_kmajor_desc(bhi + KP * 128);
      const bool last = (pos + 1 == flush) || (t == nblk - 1);
      if (LB && elect_one()) {
        const uint32_t idesc_b = idesc_bf16_m128(KP);
        const uint32_t bbf = bhi + 2 * KP * 128;  // bf16(B), interleaved K-major
#pragma unroll
        for (int o = 0; o < ((RTD && (p.debug & 1)) ? 0 : NOUT); ++o) {
          const uint32_t dt = tbase + ab * NACC + o * KP;
          const uint32_t ahi = tbase + abase + a * ASTAGE + o * OCOLS;
#pragma unroll
          for (int kk = 0; kk < BJ / 8; ++kk) {
            mma_tf32_ts(dt, ahi + 8 * kk, dhi + 2 * kk, idesc, (pos > 0 || kk > 0) ? 1u : 0u);
            mma_tf32_ts(dt, ahi + 8 * kk, dlo + 2 * kk, idesc, 1u);
          }
#pragma unroll
          for (int k2 = 0; k2 < ((KGP_TC_INSTR && (p.debug & 8)) ? 0 : BJ / 16); ++k2)
            mma_f16_ts(dt, ahi + 32 + 8 * k2, interleave_kmajor_desc(bbf + k2 * 2 * KP * 16, KP * 16, 128), idesc_b, 1u);
        }
        tc_commit(&empty[s]);
        tc_commit(&aempty[a]);
        if (last) tc_commit(&accfull[ab]);
      } else if (SPLIT == 2 && elect_one()) {
        // bf16x3: A0 B0 + A0 B1 + A1 B0 per output and K=16 step (kind::f16)
        const uint32_t idesc_b = idesc_bf16_m128(KP);
#pragma unroll
        for (int o = 0; o < ((RTD && (p.debug & 1)) ? 0 : NOUT); ++o) {
          const uint32_t dt = tbase + ab * NACC + o * KP;
          const uint32_t a0 = tbase + abase + a * ASTAGE + o * OCOLS;
#pragma unroll
          for (int k2 = 0; k2 < BJ / 16; ++k2) {
            const uint64_t b0 = interleave_kmajor_desc(bhi + k2 * 2 * KP * 16, KP * 16, 128);
            const uint64_t b1 = interleave_kmajor_desc(bhi + 64 * KP + k2 * 2 * KP * 16, KP * 16, 128);
            mma_f16_ts(dt, a0 + 8 * k2, b0, idesc_b, (pos > 0 || k2 > 0) ? 1u : 0u);
            mma_f16_ts(dt, a0 + 8 * k2, b1, idesc_b, 1u);
            mma_f16_ts(dt, a0 + 16 + 8 * k2, b0, idesc_b, 1u);
          }
        }
        tc_commit(&empty[s]);
        tc_commit(&aempty[a]);
        if (last) tc_commit(&accfull[ab]);
      } else if (W2 && elect_one()) {
        const uint32_t idesc_w = idesc_tf32_m128(2 * KP);
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
          const uint32_t dt = tbase + ab * NACC + o * 2 * KP;
          const uint32_t ahi = tbase + abase + (a * ATILES + o * TPO) * 32;
#pragma unroll
          for (int kk = 0; kk < BJ / 8; ++kk) {
            mma_tf32_ts(dt, ahi + 8 * kk, dhi + 2 * kk, idesc_w, (pos > 0 || kk > 0) ? 1u : 0u);  // hi [B_hi | B_lo]
            mma_tf32_ts(dt, ahi + 32 + 8 * kk, dhi + 2 * kk, idesc, 1u);                           // lo B_hi
          }
        }
        tc_commit(&empty[s]);
        tc_commit(&aempty[a]);
        if (last) tc_commit(&accfull[ab]);
      } else if (!LB && !W2 && SPLIT != 2 && elect_one()) {  // (exactly one elect_one() per branch chain)
#pragma unroll
        for (int o = 0; o < ((RTD && (p.debug & 1)) ? 0 : NOUT); ++o) {
          const uint32_t dt = tbase + ab * NACC + o * KP;
          const uint32_t ahi = tbase + abase + (a * ATILES + o * TPO) * 32;
#pragma unroll
          for (int kk = 0; kk < BJ / 8; ++kk) {
            const uint32_t acc = (pos > 0 || kk > 0) ? 1u : 0u;
            mma_tf32_ts(dt, ahi + 8 * kk, dhi + 2 * kk, idesc, acc);
            if (SPLIT == 3) {
              mma_tf32_ts(dt, ahi + 8 * kk, dlo + 2 * kk, idesc, 1u);
              mma_tf32_ts(dt, ahi + 32 + 8 * kk, dhi + 2 * kk, idesc, 1u);
            }
          }
        }
        tc_commit(&empty[s]);
        tc_commit(&aempty[a]);
        if (last) tc_commit(&accfull[ab]);
      }
      __syncwarp();
      KGP_TR(8, t);
      if (last) {
        pos = 0;
        if (++ab == NAB) { ab = 0; ph_acc ^= 1; }
      } else {
        ++pos;
      }
      if (++s == NSB) { s = 0; ph_s ^= 1; }
      if (++a == NSA) { a = 0; ph_a ^= 1; }
    }
  } else if (warp == WDIST) {
    // ------------------------------------------------------------ distance MMA issuer (DMMA only)
    if (DMMA) {
      const uint32_t idesc_d = idesc_tf32_m128(BJ);
      const uint32_t vlo_off = (uint32_t)BJ * KD * 4u;
      int s = 0, db = 0;
      uint32_t ph_s = 0, ph_d = 0;
      for (int t = 0; t < nblk; ++t) {
        mbar_wait(&full[s], ph_s);
        mbar_wait(&dempty[db], ph_d ^ 1);
        tc_fence_after();
        KGP_TR(1, t);
        if (elect_one()) {
          const uint32_t va = smem_u32(sV + s * VBYTES);
          const uint32_t dd = tbase + dbase + db * BJ;
#pragma unroll
          for (int kk = 0; kk < ((KGP_TC_INSTR && (p.debug & 2)) ? 0 : KD / 8); ++kk) {
            // one K=8 step = two 16-byte chunks; chunk stride (LBO) = rows * 16 B
            const uint32_t uh = tbase + ucol + 8 * kk, ul = uh + KDS;  // U' hi / lo in TMEM
            const uint64_t vh = interleave_kmajor_desc(va + kk * 2 * BJ * 16, BJ * 16, 128);
            const uint64_t vl = interleave_kmajor_desc(va + vlo_off + kk * 2 * BJ * 16, BJ * 16, 128);
            mma_tf32_ts(dd, uh, vh, idesc_d, kk > 0 ? 1u : 0u);
            if (!KGP_TC_DIST4 || 8 * kk < D) {  // DIST4: lo parts only in the coordinate columns
              mma_tf32_ts(dd, uh, vl, idesc_d, 1u);
              mma_tf32_ts(dd, ul, vh, idesc_d, 1u);
            }
          }
          tc_commit(&dfull[t % NSET]);  // to the set that owns block t (its own phase sequence)
          if (!KGP_TC_LEAN) tc_commit(&empty[s]);  // this stage's V' has been read
        }
        __syncwarp();
        KGP_TR(2, t);
        if (++s == NSB) { s = 0; ph_s ^= 1; }
        if (++db == ND) { db = 0; ph_d ^= 1; }
      }
    }
  } else if (warp < NCW) {
    // ------------------------------------------------------------ compute warps
    // NS sets of four warps (one per TMEM lane quadrant) take blocks round-robin, so one
    // set's TMEM/barrier latencies overlap the other sets' transform work.
    const int qd = warp & 3;    // TMEM lane quadrant
    const int set = warp >> 2;  // blocks t = set (mod NS)
    const int g = lane & 3;
    // rows owned by this thread: 32 qd + lane/4 + {0, 8, 16, 24}; columns 2g + {0,1} + 8m, m < 4
    float u[4][DMMA ? 1 : D];
    float qi[4];
    if (!DMMA) {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int64_t r = (int64_t)blockIdx.x * 128 + qd * 32 + (lane >> 2) + 8 * rr;
        const bool ok = r < p.nrows;
        const float* xr = p.xrow + (ok ? r : 0) * (D + 1);
        qi[rr] = ok ? xr[0] : 0.f;
#pragma unroll
        for (int k = 0; k < (DMMA ? 1 : D); ++k) u[rr][k] = ok ? xr[1 + k] : 0.f;
      }
    }
    const uint32_t lane_base = tbase + ((uint32_t)(qd * 32) << 16);
    for (int t = set; t < nblk; t += NSET) {
      const int s = t & (NSB - 1), a = t % NSA, db = t % ND;
      const uint32_t ph_s = (t >> nsb_log) & 1, ph_a = (t / NSA) & 1;
      const uint32_t ph_e = (t / NSET) & 1;  // this set's own block count: dfull[set] phase
      if (use_ld32(NOUT, SPLIT, DMMA)) {
        // thread = row qd*32 + lane; 32x32b loads/stores of 16 columns at a time
        mbar_wait_backoff(&dfull[set], ph_e, KGP_TC_SLEEP_COMP);
        tc_fence_after();
        if (qd == 0) KGP_TR(3, t);
        uint32_t v0[16], v1[16];
        if (KGP_TC_INSTR && (p.debug & 32)) {  // diagnostic: no distance loads
#pragma unroll
          for (int i = 0; i < 16; ++i) v0[i] = v1[i] = __float_as_uint(1.0f + lane);
        } else {
          tmem_ld16(lane_base + dbase + db * BJ, v0);
          tmem_ld16(lane_base + dbase + db * BJ + 16, v1);
          tc_wait_ld_tied(v0);
          tc_wait_ld_tied(v1);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[db]);
        if (qd == 0) KGP_TR(4, t);
        // the first KGP_TC_PRE 16-column halves are transformed before the A-stage wait (off the
        // chain MMA(t - NS) -> stage free -> tile stored -> MMA(t))
        float2 kv[2][8], gv[2][8];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          if (half >= KGP_TC_PRE) continue;
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const uint32_t* vv = half ? v1 : v0;
            const float2 t2 = make_float2(__uint_as_float(vv[2 * m]), __uint_as_float(vv[2 * m + 1]));
            transform2<KT, NEED_G>(t2, kv[half][m], gv[half][m]);
          }
        }
        mbar_wait_backoff(&aempty[a], ph_a ^ 1, KGP_TC_SLEEP_COMP);
        tc_fence_after();
        if (qd == 0) KGP_TR(5, t);
        const uint32_t tcol = lane_base + abase + a * ASTAGE;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            if (half < KGP_TC_PRE) break;
            const uint32_t* vv = half ? v1 : v0;
            const float2 t2 = make_float2(__uint_as_float(vv[2 * m]), __uint_as_float(vv[2 * m + 1]));
            if (KGP_TC_INSTR && (p.debug & 4)) {
              kv[half][m] = gv[half][m] = t2;
            } else if (m < KGP_TC_EXPPOLY) {
              transform2<KT, NEED_G, true, true>(t2, kv[half][m], gv[half][m]);
            } else {
              transform2<KT, NEED_G>(t2, kv[half][m], gv[half][m]);
            }
          }
          if (KGP_TC_INSTR && (p.debug & 16)) {  // diagnostic: no A-tile stores (keep the values live)
            if (__float_as_uint(kv[half][0].x) == 0x7fc00001u && __float_as_uint(gv[half][0].y) == 0x7fc00001u) p.part[0] = 0.f;
          } else if (SPLIT == 2) {
            store_row16_bf(tcol + 8 * half, tcol + 16 + 8 * half, kv[half]);
            if (NEED_G) store_row16_bf(tcol + OCOLS + 8 * half, tcol + OCOLS + 16 + 8 * half, gv[half]);
          } else if (LB) {
            store_row16_lb(tcol + 16 * half, tcol + 32 + 8 * half, kv[half]);
            store_row16_lb(tcol + OCOLS + 16 * half, tcol + OCOLS + 32 + 8 * half, gv[half]);
          } else {
            store_row16<SPLIT>(tcol + 16 * half, kv[half]);
            if (NEED_G) store_row16<SPLIT>(tcol + TPO * 32 + 16 * half, gv[half]);
          }
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[a]);
        if (qd == 0) KGP_TR(6, t);
        continue;
      }
      float2 acc[4][4];  // [row][column pair m]: rows lane/4 + 8 rr, columns 2g + 8m + {0,1}
      if (DMMA) {
        mbar_wait(&dfull[set], ph_e);
        tc_fence_after();
        const uint32_t dcol = lane_base + dbase + db * BJ;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t v[16];
          tmem_ld_16x256b_x4(dcol + ((uint32_t)(16 * half) << 16), v);
          tc_wait_ld_tied(v);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            acc[2 * half][m] = make_float2(__uint_as_float(v[4 * m]), __uint_as_float(v[4 * m + 1]));
            acc[2 * half + 1][m] = make_float2(__uint_as_float(v[4 * m + 2]), __uint_as_float(v[4 * m + 3]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[db]);
      } else {
        mbar_wait(&full[s], ph_s);
        if (qd == 0) KGP_TR(3, t);
        // this thread's 8 columns, permuted by prep_cols into two float4 at 8g
        const float* xs = reinterpret_cast<const float*>(sV + s * VBYTES) + 8 * g;
        if (XP) {  // t2 = q_i + q_j + sum_k u_ik v_jk   (u = -2 gamma c_i, v = c_j, q = gamma |c|^2)
          const float4 qa = *reinterpret_cast<const float4*>(xs);
          const float4 qb = *reinterpret_cast<const float4*>(xs + 4);
          const float2 qj[4] = {make_float2(qa.x, qa.y), make_float2(qa.z, qa.w), make_float2(qb.x, qb.y),
                                make_float2(qb.z, qb.w)};
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
#pragma unroll
            for (int m = 0; m < 4; ++m) acc[rr][m] = __fadd2_rn(qj[m], make_float2(qi[rr], qi[rr]));
        } else {
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
#pragma unroll
            for (int m = 0; m < 4; ++m) acc[rr][m] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < (DMMA ? 1 : D); ++k) {
          const float4 va = *reinterpret_cast<const float4*>(xs + (k + 1) * BJ);
          const float4 vb = *reinterpret_cast<const float4*>(xs + (k + 1) * BJ + 4);
          const float2 vv[4] = {make_float2(va.x, va.y), make_float2(va.z, va.w), make_float2(vb.x, vb.y),
                                make_float2(vb.z, vb.w)};
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const float2 uk = make_float2(u[rr][k], u[rr][k]);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              if (XP) {
                acc[rr][m] = __ffma2_rn(uk, vv[m], acc[rr][m]);
              } else {
                const float2 dd = fsub2(vv[m], uk);
                acc[rr][m] = __ffma2_rn(dd, dd, acc[rr][m]);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (qd == 0) KGP_TR(4, t);
      mbar_wait(&aempty[a], ph_a ^ 1);
      tc_fence_after();
      if (qd == 0) KGP_TR(5, t);
      const uint32_t tcol = lane_base + abase + a * ATILES * 32;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        // 16-lane group `half`: this thread's rows lane/4 (+16 half) and lane/4 + 8
        float2 kv[2][4], gv[2][4];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            if (RTD && (p.debug & 4)) {
              kv[q][m] = gv[q][m] = acc[2 * half + q][m];
            } else {
              transform2<KT, NEED_G, DMMA || XP>(acc[2 * half + q][m], kv[q][m], gv[q][m]);
            }
          }
        const uint32_t taddr = tcol + ((uint32_t)(16 * half) << 16);
        store_tile<SPLIT>(taddr, kv);
        if (NEED_G) store_tile<SPLIT>(taddr + TPO * 32, gv);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[a]);
      if (qd == 0) KGP_TR(6, t);
    }
  } else {
    // ------------------------------------------------------------ drain + epilogue warps
    const int qd = warp & 3;
    const int row = qd * 32 + lane;
    const uint32_t lane_base = tbase + ((uint32_t)(qd * 32) << 16);
    const int nseg = (nblk + flush - 1) / flush;
    int ab = 0;
    uint32_t ph = 0;
#if KGP_TC_RACC
    if (W2) {
      // W2: per output [hi B_hi + lo B_hi | hi B_lo]; the two halves are summed here (fp32,
      // round-to-nearest) into the packed promotion sums racc[o kp + c]
      float racc[64];
      for (int seg = 0; seg < nseg; ++seg) {
        mbar_wait_backoff(&accfull[ab], ph, KGP_TC_SLEEP_DRAIN);
        tc_fence_after();
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (16 * q >= KP) continue;
            uint32_t v0[16], v1[16];
            tmem_ld16(lane_base + ab * NACC + o * 2 * KP + 16 * q, v0);
            tmem_ld16(lane_base + ab * NACC + o * 2 * KP + KP + 16 * q, v1);
            tc_wait_ld();
            tc_wait_ld_tied(v0);
            tc_wait_ld_tied(v1);
            if (o == NOUT - 1 && 16 * (q + 1) >= KP) {  // the single buffer is free once every column is in registers
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&accempty[ab]);
            }
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const float x = __uint_as_float(v0[jj]) + __uint_as_float(v1[jj]);
              float& a = racc[o * 32 + 16 * q + jj];
              a = (seg == 0) ? x : a + x;
            }
          }
        }
        if (++ab == NAB) { ab = 0; ph ^= 1; }
      }
#pragma unroll
      for (int o = 0; o < NOUT; ++o)
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < KP) sAcc[(o * KP + c) * 128 + row] = racc[o * 32 + c];
    } else
    // (two compute sets only: the three-set kernels' 608 threads leave no room for 64 more
    // registers per thread)
    if (NS <= 2 && NACC <= 64) {
      // promotion sums in registers (thread = row, <= 64 columns): no shared-memory traffic in
      // the sweep, whose LDS/STS would share the MIO queue with the MMA issue and TMEM ops
      float racc[64];
      for (int seg = 0; seg < nseg; ++seg) {
        mbar_wait_backoff(&accfull[ab], ph, KGP_TC_SLEEP_DRAIN);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t v[2][16];
#pragma unroll
          for (int q = 0; q < 2; ++q)
            if (32 * h + 16 * q < NACC) tmem_ld16(lane_base + ab * NACC + 32 * h + 16 * q, v[q]);
          tc_wait_ld();
#pragma unroll
          for (int q = 0; q < 2; ++q) tc_wait_ld_tied(v[q]);
          if (h == 1 || NACC <= 32) {
            if (h == 0 || 32 < NACC) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&accempty[ab]);
            }
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (32 * h + 16 * q < NACC) {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) {
                const float x = __uint_as_float(v[q][jj]);
                float& a = racc[32 * h + 16 * q + jj];
                a = (seg == 0) ? x : a + x;
              }
            }
          }
        }
        if (++ab == NAB) { ab = 0; ph ^= 1; }
      }
#pragma unroll
      for (int c = 0; c < 64; ++c)
        if (c < NACC) sAcc[c * 128 + row] = racc[c];
    } else
#endif
    for (int seg = 0; seg < nseg; ++seg) {
      mbar_wait_backoff(&accfull[ab], ph, KGP_TC_SLEEP_DRAIN);
      tc_fence_after();
      if (qd == 0) KGP_TR(9, seg);
      // groups of up to 64 columns: all loads of a group, one wait; the buffer is released
      // as soon as the last group is in registers, before the shared-memory adds (with one
      // accumulator buffer the MMA waits on exactly this release)
      for (int g0 = 0; g0 < NACC; g0 += 64) {
        uint32_t v[4][16];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (g0 + 16 * q < NACC) tmem_ld16(lane_base + ab * NACC + g0 + 16 * q, v[q]);
        tc_wait_ld();
#pragma unroll
        for (int q = 0; q < 4; ++q) tc_wait_ld_tied(v[q]);
        if (g0 + 64 >= NACC) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&accempty[ab]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (g0 + 16 * q >= NACC) break;
          float* dst = sAcc + (g0 + 16 * q) * 128 + row;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const float x = __uint_as_float(v[q][jj]);
            dst[jj * 128] = (seg == 0) ? x : dst[jj * 128] + x;
          }
        }
      }
      if (++ab == NAB) { ab = 0; ph ^= 1; }
    }
    // epilogue: fp64 scaling, + s B on the diagonal rows, strided writes -- or, when the
    // columns are split over grid.y, the raw fp32 partial sums for tc_reduce_kernel
    const int64_t r = (int64_t)blockIdx.x * 128 + row;
    if (p.part != nullptr) {
      if (r < p.nrows) {
        float* dst = p.part + ((int64_t)(p.slot0 + blockIdx.y) * p.nrows + r) * (NOUT * KP);
        for (int c = 0; c < NOUT * KP; ++c) dst[c] = sAcc[c * 128 + row];
      }
    } else if (r < p.nrows) {
      for (int c = 0; c < p.k; ++c) {
        const double ak = (double)sAcc[c * 128 + row];
        const int64_t o = r * p.o_rs + c * p.o_cs;
        if (p.out_k) {
          double val = p.f2 * ak;
          if (p.diag_row0 >= 0) val += p.s * p.b[(p.diag_row0 + r) * p.b_rs + c * p.b_cs];
          p.out_k[o] = val;
        }
        if (p.out_df) p.out_df[o] = p.two_f * ak;
        if (NEED_G && p.out_dl) p.out_dl[o] = p.scale_dl * (double)sAcc[(KP + c) * 128 + row];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// sum the grid.y column-split partials in split order, then the epilogue of kmm_tc_kernel
__global__ void tc_reduce_kernel(const TcParams p, int nsplit, int nacc) {
  if (p.gate != nullptr && *p.gate == 0) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.nrows * p.k) return;
  const int64_t r = e / p.k;
  const int c = (int)(e % p.k);
  double ak = 0.0, ag = 0.0;
  for (int z = 0; z < nsplit; ++z) {
    const float* src = p.part + ((int64_t)z * p.nrows + r) * nacc;
    ak += (double)src[c];
    if (nacc > p.kp) ag += (double)src[p.kp + c];
  }
  const int64_t o = r * p.o_rs + c * p.o_cs;
  if (p.out_k) {
    double val = p.f2 * ak;
    if (p.diag_row0 >= 0) val += p.s * p.b[(p.diag_row0 + r) * p.b_rs + c * p.b_cs];
    p.out_k[o] = val;
  }
  if (p.out_df) p.out_df[o] = p.two_f * ak;
  if (nacc > p.kp && p.out_dl) p.out_dl[o] = p.scale_dl * ag;
}

template <int KT, int D, int NOUT, int SPLIT, int LBM>
int launch_one(const TcParams& p_in, cudaStream_t st) {
  constexpr bool LB = (LBM == 1 || LBM == 2);
  auto kern = kmm_tc_kernel<KT, D, NOUT, SPLIT, LBM>;
  TcParams p = p_in;
  const size_t stage = (size_t)tc_rhs_block_bytes(SPLIT, LB, p.kp) + Geo<D>::VBYTES;
  const size_t fixed = Geo<D>::UBYTES + (size_t)NOUT * p.kp * 128 * 4 + 512;
  const size_t limit = 225 * 1024;
  p.nsb = (fixed + 8 * stage <= limit) ? 8 : 4;  // deeper prefetch when shared memory allows
  const size_t smem = fixed + p.nsb * stage;
  KGP_REQUIRE(smem <= limit, KGP_ERR_INVALID, "fast operator tile config needs %zu B of shared memory", smem);
  KGP_SMEM_ATTR(kern, limit);
  const int nsplit = (p.nblk - p.tbeg + p.nper - 1) / p.nper;
  dim3 grid((unsigned)((p.nrows + 127) / 128), (unsigned)nsplit);
  if (p.ev_start) KGP_CUDA(cudaEventRecord(p.ev_start, st));
  kern<<<grid, nthreads_for(ns_of(NOUT, SPLIT, LBM)), smem, st>>>(p);
  KGP_LAUNCH("kmm_tc_kernel");
  if (p.ev_stop) KGP_CUDA(cudaEventRecord(p.ev_stop, st));
  if (p.part != nullptr && !p.noreduce) {  // the partials of every slot so far, in slot order
    const int64_t cnt = p.nrows * p.k;
    tc_reduce_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(p, p.slot0 + nsplit, NOUT * p.kp);
    KGP_LAUNCH("tc_reduce_kernel");
  }
  return KGP_OK;
}

template <int KT, int D>
int launch_kt_d(const TcParams& p, int nout, int split, cudaStream_t st) {
  if (split == 2) {
    if constexpr (Geo<D>::DMMA) {
      return nout == 1 ? launch_one<KT, D, 1, 2, 0>(p, st) : launch_one<KT, D, 2, 2, 0>(p, st);
    } else {
      set_error(KGP_ERR_INVALID, "bf16x3 precision needs d > 4 (tensor-core distance)");
      return KGP_ERR_INVALID;
    }
  }
  if (nout == 1) return split == 3 ? launch_one<KT, D, 1, 3, 0>(p, st) : launch_one<KT, D, 1, 1, 0>(p, st);
  if (split != 3) return launch_one<KT, D, 2, 1, 0>(p, st);
  if (p.lb == 3) return launch_one<KT, D, 2, 3, 3>(p, st);
  if constexpr (Geo<D>::DMMA && D == 8) {
    if (p.lb == 1) return launch_one<KT, D, 2, 3, 1>(p, st);
    if (p.lb == 2) return launch_one<KT, D, 2, 3, 2>(p, st);
  }
  return launch_one<KT, D, 2, 3, 0>(p, st);
}

template <int KT>
int launch_kt(const TcParams& p, int dpad, int nout, int split, cudaStream_t st) {
  switch (dpad) {
    case 2: return launch_kt_d<KT, 2>(p, nout, split, st);
    case 4: return launch_kt_d<KT, 4>(p, nout, split, st);
    case 8: return launch_kt_d<KT, 8>(p, nout, split, st);
    case 16: return launch_kt_d<KT, 16>(p, nout, split, st);
  }
  set_error(KGP_ERR_INVALID, "fast path supports d <= 16");
  return KGP_ERR_INVALID;
}

}  // namespace

int tc_pad_dim(int d) { return d <= 2 ? 2 : d <= 4 ? 4 : d <= 8 ? 8 : 16; }
bool tc_direct(int dpad) { return dpad <= KGP_TC_DMIN; }
int tc_dist_mode(int dpad) { return dpad <= KGP_TC_DMIN ? 0 : (KGP_TC_XP ? 2 : 1); }

int tc_col_block_bytes(int dpad) {
  if (tc_dist_mode(dpad) != 1) return (dpad + 1) * BJ * 4;
  const int kd = tc_dist_kd(dpad);
  return 2 * BJ * kd * 4;
}

static int tc_fixed_cols(int dpad, int ns) {
  if (tc_dist_mode(dpad) != 1) return 0;
  const int kd = tc_dist_kd(dpad);
  return ns * BJ + 2 * ((kd + 15) / 16 * 16);  // distance buffers + U' hi/lo
}

// RHS columns per launch with `nab` accumulator buffers: TMEM holds nab x nout x kp
// accumulator columns + distance buffers + U' + NS A stages
int tc_max_kp(int dpad, int nout, int split, int nab) {
  const int ns = ns_for(nout, split);
  const int stage = nout * (split == 3 ? 2 : 1) * 32;
  int kp = (512 - tc_fixed_cols(dpad, ns) - ns * stage) / (nab * nout);
  kp = kp / 16 * 16;
  if (kp > 128) kp = 128;
  // shared memory (launch_one): fp32 promotion sums + at least a 4-deep operand ring
  const int tpo = split == 3 ? 2 : 1;
  while (kp > 16 && (size_t)nout * kp * 128 * 4 + 512 + 4 * ((size_t)tpo * kp * 128 + tc_col_block_bytes(dpad)) >
                        225 * 1024)
    kp -= 16;
  return kp;
}

int tc_nsa(int, int nout, int split, int) { return ns_for(nout, split); }

// LB layout for the fused two-output 3xTF32 product with the tensor-core distance at
// dpad = 8 (U' takes 2 x 16 columns): TMEM holds nab x 2 x kp accumulators (nab kp <= 64),
// two distance buffers, U' and three 96-column A stages: 2 nab kp + 64 + 32 + 288 <= 512.
// Used for 32 < kp <= 64 (one accumulator buffer), where it measured faster (n = 65536,
// k = 64: 5.83 -> 5.24 ms); at kp <= 32 it ties (k = 32: 3.40 ms both) or loses (k = 16:
// 3.05 -> 3.24 ms), so the all-tf32 two-stage layout stays there. Env KGP_TC_LB=0 disables
// it, KGP_TC_LB=2 forces it for every kp <= 64.
//
// LB mode 2 (kp <= 32): three compute sets, three A stages and two distance buffers;
// TMEM = 2 nab kp + 64 + 32 + 288 <= 512: two accumulator buffers up to kp = 32.
// Measured at cfg2 shape (k = 32): 3.45 ms against 3.39 for the classic layout, so it is
// off by default (env KGP_TC_LB3=1 selects it).
int tc_lb_mode(int dpad, int nout, int split, int kp) {
  static const int env = [] {
    const char* s = getenv("KGP_TC_LB");
    return s ? atoi(s) : 1;
  }();
  static const int env3 = [] {
    const char* s = getenv("KGP_TC_LB3");
    return s ? atoi(s) : 0;
  }();
  static const int envw = [] {
    const char* s = getenv("KGP_TC_W2");
    return s ? atoi(s) : 0;
  }();
  // W2 measured (n = 65536, two outputs): Gaussian d=8 k=32 3.02 -> 3.15 ms (the single accumulator
  // buffer's drain stalls; with flush 16 3.06), k=16 2.54 -> 2.38; Matern-3/2 d=4 k=16 4.21 ->
  // 5.06. Operator error 3.05e-6 -> 2.52e-6 (the hi B_lo column sums promoted separately). Off by
  // default (env KGP_TC_W2=1): the MMA issue count is not what bounds the kernel at k = 32.
  if (envw && nout == 2 && split == 3 && kp <= 32 && !env3) return 3;
  if (env == 0 || tc_dist_mode(dpad) != 1 || dpad != 8 || nout != 2 || split != 3 || kp > 64) return 0;
  if (kp > 32) return 1;
  if (env3) return 2;
  return env == 2 ? 1 : 0;
}

// TMEM accumulator buffers for a LB mode (0: the caller's choice for the classic layout)
int tc_lb_nab(int mode, int kp) {
  if (mode == 3) return 1;  // W2: 2 x 2kp accumulator columns, one buffer
  if (mode == 2) return kp <= 32 ? 2 : 1;
  if (mode == 1) return kp <= 32 ? 2 : 1;
  return 0;
}

// bytes of one 32-row RHS block in bsplit: tf32 hi (| lo) K-major 128B-swizzled (| bf16 interleaved)
int tc_rhs_block_bytes(int split, bool lb, int kp) { return ((split == 3 ? 2 : 1) * 128 + (lb ? 64 : 0)) * kp; }
// (split 2, bf16x3: B0 | B1 as bf16, 2 x 64 kp bytes = the same 128 kp as one tf32 tile)

// Column split factor that fills the last wave of 148 SMs (1 CTA/SM): the smallest
// S <= maxsplit reaching 95% wave efficiency with >= 16 column blocks per CTA.
int tc_col_split(int64_t nrows, int nblk, int maxsplit) {
  const int64_t rb = (nrows + 127) / 128;
  int best = 1;
  double best_eff = 0.0;
  for (int sp = 1; sp <= maxsplit; ++sp) {
    if (sp > 1 && nblk / sp < 16) break;
    const int64_t units = rb * sp;
    const double eff = (double)units / (double)(((units + 147) / 148) * 148);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = sp;
    }
    if (eff >= 0.95) break;
  }
  return best;
}

int launch_kmm_tc(int kt, int dpad, int nout, int split, const TcParams& p, cudaStream_t st) {
  switch (kt) {
    case GAUSS: return launch_kt<GAUSS>(p, dpad, nout, split, st);
    case MAT32: return launch_kt<MAT32>(p, dpad, nout, split, st);
    case MAT52: return launch_kt<MAT52>(p, dpad, nout, split, st);
  }
  set_error(KGP_ERR_INVALID, "unknown kernel id %d", kt);
  return KGP_ERR_INVALID;
}

}  // namespace kgp
