// Fused kernel-matrix MatMul in fp64 (precision KGP_FP64): the parity anchor.
//
// Same contract as KernelEngine._streamed_matmul (kmat.py:165-189): per entry a
// direct-difference r^2 in fp64 (_panels_numba.py:23-34 order, no FMA
// contraction), the kernel and its l-derivative (_panels_numba.py:37-131),
// contracted against the RHS block in fp64. Khat is never stored, not even a tile:
//
// one thread = one row. A CTA of 128 threads stages a tile of TJ column points and the
// matching RHS rows in shared memory; every thread evaluates kappa (and dkappa/dl) of its
// row against each column and FMAs it straight into its KS register accumulators (the
// column data are warp-broadcast reads). The RHS is processed in slices of KS <= 28/48
// columns (grid.y); the column range is split over grid.z so that the CTAs fill whole waves
// of the instantiation's real occupancy, and the partial sums are reduced in a fixed order
// (deterministic). Three kernels share this contract:
//   kmm_f64_kernel        one lane per row (narrow slices);
//   kmm_f64_split_kernel  2 or 4 lanes per row share every kernel-entry evaluation and split the
//                         slice's columns (wide slices: one evaluation per entry for up to 64
//                         columns instead of one per 16..28-column slice);
//   kmm_f64_sym_kernel    the square operator with <= 4 columns evaluates each entry once for
//                         both triangles.
// Bound: the FP64 pipe (distance 3d + exp 13 + KS FMA per entry and output; the exponential is
// exp_neg64t, kgp_common.cuh).
#include <stdlib.h>

#include <map>
#include <mutex>
#include <utility>

#include "kgp_common.cuh"
#include "kgp_internal.h"

#ifndef KGP_F64_FASTEXP
#define KGP_F64_FASTEXP 1  // the operator's entries through exp_neg64 (kgp_common.cuh)
#endif
#ifndef KGP_F64_SYM_FG
#define KGP_F64_SYM_FG 0  // symmetric small-k kernel: exp_neg64 for the Gaussian (measured: configs[0] OTF eval 4.99 -> 5.08 ms, off)
#endif
#ifndef KGP_F64_CAP2
// RHS columns per slice with two outputs (register budget): 28 -> 168 registers, 3 CTAs per SM;
// measured against 24 (n = 16384): Gaussian d=8 k=51 9.67 -> 5.03 ms (two slices of 28 instead of
// three of 20: each slice re-evaluates every kernel entry), Matern-5/2 d=2 k=28 3.89 -> 2.53 ms;
// 32 (211 registers, 2 CTAs per SM) made cfg2's k = 32 55.9 -> 93.6 ms, so 32 runs as 2 x 16
#define KGP_F64_CAP2 28
#endif
#ifndef KGP_F64_SWP
#define KGP_F64_SWP 0  // 1: one-lane kernel evaluates entry jj + 1 while contracting entry jj (measured, off)
#endif
#ifndef KGP_F64_FMADIST
#define KGP_F64_FMADIST 0  // 1: r^2 accumulated with FMA (one rounding per term fewer than numba's order)
#endif
#if KGP_F64_FMADIST
#define KGP_R2ACC(r2, df) fma((df), (df), (r2))
#else
#define KGP_R2ACC(r2, df) __dadd_rn((r2), __dmul_rn((df), (df)))  // numba's rounding (no FMA contraction)
#endif
#if KGP_F64_FASTEXP
#define KGP_KAPPA kappa64f
#define KGP_DKAPPA dkappa64f
#else
#define KGP_KAPPA kappa64
#define KGP_DKAPPA dkappa64
#endif

namespace kgp {

namespace {

constexpr int NT = 128;  // threads = rows per CTA
constexpr int TJ = 64;   // columns per shared-memory tile
constexpr int MAXD = 16;

template <int KT, int NOUT, int KS, int DB>
__global__ void __launch_bounds__(NT) kmm_f64_kernel(const F64Params p) {
  if (p.gate != nullptr && *p.gate == 0) return;  // PCG iteration past convergence
  __shared__ double sXj[TJ][DB + 1];
  __shared__ __align__(16) double sB[TJ][KS];
  __shared__ double sTab[64];  // 2^(j/64) of exp_neg64t (visible after the first tile barrier)
  exp_tab_fill(sTab);

  const int tid = threadIdx.x;
  const int64_t r = (int64_t)blockIdx.x * NT + tid;
  const int c0 = blockIdx.y * KS;  // RHS slice
  const int d = p.d;
  const int64_t jb = (int64_t)blockIdx.z * p.jchunk;
  const int64_t je = jb + p.jchunk < p.ncols ? jb + p.jchunk : p.ncols;
  const bool live = r < p.nrows;

  double xi[DB];  // DB: d rounded up to 4, 8 or 16 (register budget)
#pragma unroll
  for (int q = 0; q < DB; ++q) xi[q] = (live && q < d) ? p.xr[r * d + q] : 0.0;
  double acc[KS], accg[NOUT == 2 ? KS : 1];
#pragma unroll
  for (int c = 0; c < KS; ++c) {
    acc[c] = 0.0;
    if (NOUT == 2) accg[c] = 0.0;
  }

  // EB entries per inner step (independent distance / exponential chains, the contraction after
  // them in column order so every sum keeps its order). Measured at EB = 4 / 2 over k = 4..64,
  // d = 3..8 (tools/f64_grid.py): 25-35 % faster for one output at d = 8, k = 16..18 and 32..34,
  // but 15-60 % slower for two outputs and for k = 24..28 and 40..48 (the chains' registers cost
  // a resident CTA); configs[0] eval 4.93 -> 5.10 ms. One entry per step stays.
  constexpr int EB = 1;
  static_assert(TJ % EB == 0, "entry batch");
  for (int64_t j0 = jb; j0 < je; j0 += TJ) {
    const int nj = (int)(je - j0 < TJ ? je - j0 : TJ);
    const int nje = (nj + EB - 1) / EB * EB;  // rows past nj up to the batch boundary: zero RHS
    __syncthreads();
    for (int e = tid; e < nj * d; e += NT) sXj[e / d][e % d] = p.xc[(j0 + e / d) * d + e % d];
    for (int e = tid; e < nje * KS; e += NT) {
      const int jj = e / KS, c = e % KS;
      const int cc = c0 + c;
      sB[jj][c] = (jj < nj && cc < p.k) ? p.b[(j0 + jj) * p.b_rs + (int64_t)cc * p.b_cs] : 0.0;
    }
    __syncthreads();
#if KGP_F64_SWP
    // software pipeline: entry jj + 1 is evaluated in the same loop body that contracts entry jj,
    // so the in-order warp has the independent FMA stream to issue while the distance /
    // exponential chain waits on its latencies (two live values more, no extra accumulators)
    auto eval = [&](int jm, double& kvo, double& gvo) {
      double r2 = 0.0;
#pragma unroll
      for (int q = 0; q < DB; ++q) {
        if (q < d) {
          const double df = xi[q] - sXj[jm][q];
          r2 = KGP_R2ACC(r2, df);  // numba's rounding (no FMA contraction)
        }
      }
      gvo = 0.0;
      if (NOUT == 2) {
        kd64f<KT, (DB >= 8)>(r2, p.l, kvo, gvo, sTab);  // one exponential for both outputs
      } else {
        kvo = kappa64f<KT, (DB >= 8)>(r2, p.l, sTab);
      }
    };
    double kc, gc;
    eval(0, kc, gc);
    for (int jj = 0; jj < nj; ++jj) {
      double kn, gn;
      eval(jj + 1 < nj ? jj + 1 : nj - 1, kn, gn);  // the last one is not used
#pragma unroll
      for (int c = 0; c < KS; c += 2) {
        const double2 bv = *reinterpret_cast<const double2*>(&sB[jj][c]);
        acc[c] = fma(kc, bv.x, acc[c]);
        acc[c + 1] = fma(kc, bv.y, acc[c + 1]);
        if (NOUT == 2) {
          accg[c] = fma(gc, bv.x, accg[c]);
          accg[c + 1] = fma(gc, bv.y, accg[c + 1]);
        }
      }
      kc = kn;
      gc = gn;
    }
#else
    for (int jj = 0; jj < nje; jj += EB) {
      double kv[EB], gv[EB];
#pragma unroll
      for (int u = 0; u < EB; ++u) {
        const int jm = jj + u < nj ? jj + u : nj - 1;  // past nj: any finite value (its RHS row is 0)
        double r2 = 0.0;
#pragma unroll
        for (int q = 0; q < DB; ++q) {
          if (q < d) {
            const double df = xi[q] - sXj[jm][q];
            r2 = KGP_R2ACC(r2, df);  // numba's rounding (no FMA contraction)
          }
        }
        gv[u] = 0.0;
#if KGP_F64_FASTEXP
        if (NOUT == 2) {
          kd64f<KT, (DB >= 8)>(r2, p.l, kv[u], gv[u], sTab);  // one exponential for both outputs
        } else {
          kv[u] = kappa64f<KT, (DB >= 8)>(r2, p.l, sTab);
        }
#else
        kv[u] = KGP_KAPPA<KT>(r2, p.l);
        if (NOUT == 2) gv[u] = KGP_DKAPPA<KT>(r2, p.l);
#endif
      }
#pragma unroll
      for (int u = 0; u < EB; ++u) {
#pragma unroll
        for (int c = 0; c < KS; c += 2) {
          const double2 bv = *reinterpret_cast<const double2*>(&sB[jj + u][c]);
          acc[c] = fma(kv[u], bv.x, acc[c]);
          acc[c + 1] = fma(kv[u], bv.y, acc[c + 1]);
          if (NOUT == 2) {
            accg[c] = fma(gv[u], bv.x, accg[c]);
            accg[c + 1] = fma(gv[u], bv.y, accg[c + 1]);
          }
        }
      }
    }
#endif
  }
  if (!live) return;
  // epilogue (kmat.py:186-188): scale, + s B on the diagonal rows; raw partials when split
#pragma unroll
  for (int c = 0; c < KS; ++c) {
    const int cc = c0 + c;
    if (cc >= p.k) continue;
    if (p.part) {
      const int64_t slot = ((int64_t)blockIdx.z * p.nrows + r) * p.k + cc;
      p.part[slot] = acc[c];
      if (NOUT == 2) p.part[p.part_stride + slot] = accg[c];
      continue;
    }
    const int64_t o = r * p.o_rs + (int64_t)cc * p.o_cs;
    if (p.out_k) {
      double v = p.f2 * acc[c];
      if (p.diag_row0 >= 0) v += p.s * p.b[(p.diag_row0 + r) * p.b_rs + (int64_t)cc * p.b_cs];
      p.out_k[o] = v;
    }
    if (p.out_df) p.out_df[o] = p.two_f * acc[c];
    if (NOUT == 2 && p.out_dl) p.out_dl[o] = p.f2_dl * accg[c];
  }
}

// ------------------------------------------------------------------ lane-split wide-k path
// Every RHS slice of kmm_f64_kernel re-evaluates the kernel entries (distance + exponential, ~40
// of the ~70 FP64 instructions per entry and slice at 16 columns and two outputs), and the slice
// width is capped by the accumulator registers. Here G = 2 or 4 adjacent lanes share a row: lane
// h of the group evaluates every G-th entry of the row (one evaluation per entry in all), the
// group exchanges kappa (and dkappa/dl) by width-G shuffles, and each lane contracts all the
// entries against ITS KQ columns of the slice -- G x KQ columns per evaluation with KQ
// accumulators per lane and output (k = 32 with two outputs: one pass instead of 2 x 16).
// Each (row, column) sum runs over the entries in the same order as in kmm_f64_kernel with
// the same kappa, so both kernels give the same bits.
constexpr int NTS = 256;  // threads per CTA (NTS / G rows)
constexpr int kqp_of(int kq, int g) {
  // padded lane stride of a column tile row: the G sub-rows a warp reads at once (16-byte loads)
  // must fall into different 16-byte bank groups of the 128-byte bank row
  int q = kq;
  for (;; q += 2) {
    bool ok = true;
    for (int a = 0; a < g; ++a)
      for (int b = a + 1; b < g; ++b) ok = ok && ((q * 8 * (b - a)) % 128 >= 16) && ((q * 8 * (b - a)) % 128 <= 112);
    if (ok) return q;
  }
}

template <int KT, int NOUT, int KQ, int DB, int G>
__global__ void __launch_bounds__(NTS, (NOUT * KQ <= 32) ? 2 : 1) kmm_f64_split_kernel(const F64Params p) {
  static_assert(KQ % 2 == 0 && (G == 2 || G == 4), "lane-split layout");
  if (p.gate != nullptr && *p.gate == 0) return;
  constexpr int ROWS = NTS / G, KS = G * KQ, KQP = kqp_of(KQ, G);
  constexpr int EBS = 1;  // evaluation chains per lane and step (2: within 2 % either way, small spills)
  static_assert(TJ % (G * EBS) == 0, "entry batch");
  __shared__ double sXj[TJ][DB + 1];
  __shared__ __align__(16) double sB[TJ][G][KQP];
  __shared__ double sTab[64];
  exp_tab_fill(sTab);

  const int tid = threadIdx.x, h = tid % G;
  const int64_t r = (int64_t)blockIdx.x * ROWS + tid / G;
  const int c0 = blockIdx.y * KS;
  const int d = p.d;
  const int64_t jb = (int64_t)blockIdx.z * p.jchunk;
  const int64_t je = jb + p.jchunk < p.ncols ? jb + p.jchunk : p.ncols;
  const bool live = r < p.nrows;

  double xi[DB];
#pragma unroll
  for (int q = 0; q < DB; ++q) xi[q] = (live && q < d) ? p.xr[r * d + q] : 0.0;
  double acc[KQ], accg[NOUT == 2 ? KQ : 1];
#pragma unroll
  for (int c = 0; c < KQ; ++c) {
    acc[c] = 0.0;
    if (NOUT == 2) accg[c] = 0.0;
  }

  for (int64_t j0 = jb; j0 < je; j0 += TJ) {
    const int nj = (int)(je - j0 < TJ ? je - j0 : TJ);
    const int njg = (nj + G * EBS - 1) / (G * EBS) * (G * EBS);  // rows past nj up to the batch boundary: zero RHS
    __syncthreads();
    for (int e = tid; e < nj * d; e += NTS) sXj[e / d][e % d] = p.xc[(j0 + e / d) * d + e % d];
    for (int e = tid; e < njg * KS; e += NTS) {
      const int jj = e / KS, c = e % KS;
      const int cc = c0 + c;
      sB[jj][c / KQ][c % KQ] = (jj < nj && cc < p.k) ? p.b[(j0 + jj) * p.b_rs + (int64_t)cc * p.b_cs] : 0.0;
    }
    __syncthreads();
    for (int jj = 0; jj < njg; jj += G * EBS) {
      // this lane's entries of the batch: columns jj + u G + h (past nj: any finite value, the
      // RHS row is 0); EBS independent evaluation chains per lane
      double kv[EBS], gv[EBS];
#pragma unroll
      for (int u = 0; u < EBS; ++u) {
        const int jm = jj + u * G + h < nj ? jj + u * G + h : nj - 1;
        double r2 = 0.0;
#pragma unroll
        for (int q = 0; q < DB; ++q) {
          if (q < d) {
            const double df = xi[q] - sXj[jm][q];
            r2 = KGP_R2ACC(r2, df);  // numba's rounding (no FMA contraction)
          }
        }
        gv[u] = 0.0;
        if (NOUT == 2) {
          kd64f<KT, (DB >= 8)>(r2, p.l, kv[u], gv[u], sTab);
        } else {
          kv[u] = kappa64f<KT, (DB >= 8)>(r2, p.l, sTab);
        }
      }
#pragma unroll
      for (int u = 0; u < EBS; ++u) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const double kg = __shfl_sync(0xffffffffu, kv[u], g, G);
          const double gg = NOUT == 2 ? __shfl_sync(0xffffffffu, gv[u], g, G) : 0.0;
#pragma unroll
          for (int c = 0; c < KQ; c += 2) {
            const double2 bv = *reinterpret_cast<const double2*>(&sB[jj + u * G + g][h][c]);
            acc[c] = fma(kg, bv.x, acc[c]);
            acc[c + 1] = fma(kg, bv.y, acc[c + 1]);
            if (NOUT == 2) {
              accg[c] = fma(gg, bv.x, accg[c]);
              accg[c + 1] = fma(gg, bv.y, accg[c + 1]);
            }
          }
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int c = 0; c < KQ; ++c) {
    const int cc = c0 + h * KQ + c;
    if (cc >= p.k) continue;
    if (p.part) {
      const int64_t slot = ((int64_t)blockIdx.z * p.nrows + r) * p.k + cc;
      p.part[slot] = acc[c];
      if (NOUT == 2) p.part[p.part_stride + slot] = accg[c];
      continue;
    }
    const int64_t o = r * p.o_rs + (int64_t)cc * p.o_cs;
    if (p.out_k) {
      double v = p.f2 * acc[c];
      if (p.diag_row0 >= 0) v += p.s * p.b[(p.diag_row0 + r) * p.b_rs + (int64_t)cc * p.b_cs];
      p.out_k[o] = v;
    }
    if (p.out_df) p.out_df[o] = p.two_f * acc[c];
    if (NOUT == 2 && p.out_dl) p.out_dl[o] = p.f2_dl * accg[c];
  }
}

// ------------------------------------------------------------------ symmetric small-k path
// Khat is symmetric, so for the SQUARE operator with few right-hand sides (the PCG w-solve's
// single column, where evaluating kernel entries is nearly all the work) every entry is
// evaluated once: a CTA takes a pair of 128-point blocks (I, J >= I) and uses each kappa_ij for
// both y_I += K_IJ B_J (thread = row i, register accumulators) and y_J += K_IJ^T B_I (each
// warp's 32 row contributions per column j summed by a transpose-butterfly: 31 shuffles per
// 32 columns, lane l ending with column l; the warps combined in shared memory). Every
// row receives exactly one partial per partner block; P[partner][row][c] is summed in
// partner order by f64_sym_reduce_kernel (run-to-run deterministic). 64-point blocks: the
// kernel is FP64-latency-bound (ncu: fp64 pipe 49 %, stall_wait dominant at 128-point blocks
// and ~14 warps per SM), so twice the CTAs matter more than the larger tiles' reuse.
#ifndef KGP_F64_SB
#define KGP_F64_SB 64
#endif
// Butterfly chunk (columns evaluated before each transpose-sum) and the resident CTAs per SM the
// register allocation must allow. 32 columns per chunk held 32 kappa values per lane: 96 registers,
// 10 CTAs per SM, so configs[0]'s 2080 block pairs ran 1.41 waves (ncu: the second wave 41 % full).
// 4 columns and a 64-register cap (16 CTAs per SM: one wave): one-column product 61 -> 50 us at
// n = 4096, 0.82 -> 0.53 ms at n = 16384, configs[0] eval 4.93 -> 4.73 ms. Measured around it
// (tools/gpu_sym.sh): chunk 8 / 16 at 16 CTAs 50 / 56 us, chunk 8 at 20 / 24 CTAs 52 / 53 us (k = 4
// at n = 16384 0.83 -> 1.14 / 1.32 ms), chunk 4 at 24 CTAs 56 us.
#ifndef KGP_F64_SYM_Q
#define KGP_F64_SYM_Q 4
#endif
#ifndef KGP_F64_SYM_MINB
#define KGP_F64_SYM_MINB 16
#endif
constexpr int SB = KGP_F64_SB;  // points per block (64: twice the CTAs of 128, the kernel is latency-bound)
constexpr int SNW = SB / 32;    // warps per CTA

template <int KT, int KS, int DB>
__global__ void __launch_bounds__(SB, KGP_F64_SYM_MINB) kmm_f64_sym_kernel(const F64Params p, int nb, double* __restrict__ part) {
  if (p.gate != nullptr && *p.gate == 0) return;
  __shared__ double sX[SB][DB + 1];
  __shared__ double sB[SB][KS];
  __shared__ double sCol[SNW][SB][KS];
  __shared__ double sTab[64];
  exp_tab_fill(sTab);
  // tile pair (I, J), I <= J, from the linear index
  const int64_t tix = blockIdx.x;
  int I = (int)((sqrt(8.0 * (double)tix + 1.0) - 1.0) * 0.5);  // row of the packed upper triangle
  while ((int64_t)I * (I + 1) / 2 > tix) --I;
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tix) ++I;
  // packed order by J: tix = J (J + 1) / 2 + I' with I' <= J
  const int J = I;
  const int Ip = (int)(tix - (int64_t)J * (J + 1) / 2);
  const int rowblk = Ip, colblk = J;  // rowblk <= colblk
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)p.ncols, d = p.d;
  const int64_t r = (int64_t)rowblk * SB + tid;
  const bool live = r < n;
  double xi[DB];
#pragma unroll
  for (int q = 0; q < DB; ++q) xi[q] = (live && q < d) ? p.xr[r * d + q] : 0.0;
  double bi[KS];
#pragma unroll
  for (int c = 0; c < KS; ++c) bi[c] = (live && c < p.k) ? p.b[r * p.b_rs + (int64_t)c * p.b_cs] : 0.0;
  const int64_t j0 = (int64_t)colblk * SB;
  const int nj = (int)(n - j0 < SB ? n - j0 : SB);
  for (int e = tid; e < nj * d; e += SB) sX[e / d][e % d] = p.xc[(j0 + e / d) * d + e % d];
  for (int e = tid; e < SB * KS; e += SB) {  // rows past the last point stay zero
    const int jj = e / KS, c = e % KS;
    sB[jj][c] = (jj < nj && c < p.k) ? p.b[(j0 + jj) * p.b_rs + (int64_t)c * p.b_cs] : 0.0;
  }
  __syncthreads();
  const bool offdiag = rowblk != colblk;
  double acc[KS];
#pragma unroll
  for (int c = 0; c < KS; ++c) acc[c] = 0.0;
  // columns per butterfly chunk: Q x KS <= 32 values per lane (the halving steps cost Q - 1
  // shuffle-adds per Q columns whatever Q is; a smaller chunk holds fewer values in registers)
  constexpr int Q = (32 / KS < KGP_F64_SYM_Q) ? 32 / KS : KGP_F64_SYM_Q;
  for (int jc = 0; jc < SB; jc += Q) {
    double v[Q][KS];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int jj = jc + q;
      double kv = 0.0;
      if (live && jj < nj) {
        double r2 = 0.0;
#pragma unroll
        for (int t = 0; t < DB; ++t) {
          if (t < d) {
            const double df = xi[t] - sX[jj][t];
            r2 = KGP_R2ACC(r2, df);  // numba's rounding (no FMA contraction)
          }
        }
        kv = kappa64f<KT, KGP_F64_SYM_FG>(r2, p.l, sTab);
      }
#pragma unroll
      for (int c = 0; c < KS; ++c) {
        acc[c] = fma(kv, sB[jj < SB ? jj : 0][c], acc[c]);
        v[q][c] = kv * bi[c];
      }
    }
    if (offdiag) {
      // transpose-butterfly over the Q columns (log2 Q halving steps), then a plain xor-sum
      // over the lanes sharing lane % Q: lane l ends with the warp's sum for column l % Q
#pragma unroll
      for (int c = 0; c < KS; ++c) {
#pragma unroll
        for (int off = Q / 2; off >= 1; off >>= 1) {
#pragma unroll
          for (int q = 0; q < off; ++q) {
            const bool up = (lane & off) != 0;
            const double send = up ? v[q][c] : v[q + off][c];
            const double keep = up ? v[q + off][c] : v[q][c];
            v[q][c] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
#pragma unroll
        for (int off = Q; off < 32; off <<= 1) v[0][c] += __shfl_xor_sync(0xffffffffu, v[0][c], off);
        if (lane < Q) sCol[warp][jc + lane][c] = v[0][c];
      }
    }
  }
  // row direction: this block pair's contribution to rows of rowblk, partner = colblk
  if (live) {
#pragma unroll
    for (int c = 0; c < KS; ++c)
      if (c < p.k) part[((int64_t)colblk * n + r) * p.k + c] = acc[c];
  }
  if (offdiag) {  // column direction: contribution to rows of colblk, partner = rowblk
    __syncthreads();
    if (tid < nj) {
#pragma unroll
      for (int c = 0; c < KS; ++c) {
        if (c >= p.k) continue;
        double t = sCol[0][tid][c];
#pragma unroll
        for (int w = 1; w < SNW; ++w) t += sCol[w][tid][c];
        part[((int64_t)rowblk * n + j0 + tid) * p.k + c] = t;
      }
    }
  }
}

// Partial-sum reduction, RW warps per 32 consecutive elements: warp w sums the slots q = w (mod
// RW) in slot order (four loads in flight), then the RW warp sums are added in warp order --
// a fixed tree, so run-to-run identical. (One thread per element serialised 64 dependent adds
// over 16 CTAs at configs[0]: 10.6 us per product; latency, not bandwidth.)
constexpr int RW = 8;
KGP_DEV double reduce_slots(const double* __restrict__ part, int nslot, int64_t stride, int64_t e, bool live,
                            double (*red)[32]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a = 0.0;
  if (live) {
    int q = w;
    for (; q + 3 * RW < nslot; q += 4 * RW) {
      const double t0 = part[(int64_t)q * stride + e], t1 = part[(int64_t)(q + RW) * stride + e];
      const double t2 = part[(int64_t)(q + 2 * RW) * stride + e], t3 = part[(int64_t)(q + 3 * RW) * stride + e];
      a += t0;
      a += t1;
      a += t2;
      a += t3;
    }
    for (; q < nslot; q += RW) a += part[(int64_t)q * stride + e];
  }
  red[w][lane] = a;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
#pragma unroll
    for (int u = 0; u < RW; ++u) t += red[u][lane];
  }
  return t;
}

__global__ void __launch_bounds__(RW * 32) f64_sym_reduce_kernel(const F64Params p, int nb, const double* __restrict__ part) {
  if (p.gate != nullptr && *p.gate == 0) return;
  __shared__ double red[RW][32];
  const int64_t e = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t n = p.ncols;
  const bool live = e < n * p.k;
  const double a = reduce_slots(part, nb, n * p.k, e, live, red);
  if (!live || threadIdx.x >= 32) return;
  const int64_t r = e / p.k;
  const int c = (int)(e % p.k);
  const int64_t o = r * p.o_rs + (int64_t)c * p.o_cs;
  if (p.out_k) p.out_k[o] = p.f2 * a + p.s * p.b[r * p.b_rs + (int64_t)c * p.b_cs];
  if (p.out_df) p.out_df[o] = p.two_f * a;
}

template <int KT, int KS>
int launch_sym_ks(const F64Params& p, int nb, double* part, cudaStream_t st) {
  const unsigned pairs = (unsigned)((int64_t)nb * (nb + 1) / 2);
  if (p.d <= 4) kmm_f64_sym_kernel<KT, KS, 4><<<pairs, SB, 0, st>>>(p, nb, part);
  else if (p.d <= 8) kmm_f64_sym_kernel<KT, KS, 8><<<pairs, SB, 0, st>>>(p, nb, part);
  else kmm_f64_sym_kernel<KT, KS, 16><<<pairs, SB, 0, st>>>(p, nb, part);
  KGP_LAUNCH("kmm_f64_sym_kernel");
  return KGP_OK;
}

template <int KT>
int launch_sym(const F64Params& p, int nb, double* part, cudaStream_t st) {
  if (p.k == 1) return launch_sym_ks<KT, 1>(p, nb, part, st);
  if (p.k == 2) return launch_sym_ks<KT, 2>(p, nb, part, st);
  return launch_sym_ks<KT, 4>(p, nb, part, st);
}

// sum the column-split partials in split order, then the epilogue
__global__ void __launch_bounds__(RW * 32) f64_reduce_kernel(const F64Params p, int nsplit) {
  if (p.gate != nullptr && *p.gate == 0) return;
  __shared__ double red[RW][32];
  const int64_t e = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  const bool live = e < p.nrows * p.k;
  const double a = reduce_slots(p.part, nsplit, p.nrows * p.k, e, live, red);
  double g = 0.0;
  if (p.out_dl) {
    __syncthreads();
    g = reduce_slots(p.part + p.part_stride, nsplit, p.nrows * p.k, e, live, red);
  }
  if (!live || threadIdx.x >= 32) return;
  const int64_t r = e / p.k;
  const int c = (int)(e % p.k);
  const int64_t o = r * p.o_rs + (int64_t)c * p.o_cs;
  if (p.out_k) {
    double v = p.f2 * a;
    if (p.diag_row0 >= 0) v += p.s * p.b[(p.diag_row0 + r) * p.b_rs + (int64_t)c * p.b_cs];
    p.out_k[o] = v;
  }
  if (p.out_df) p.out_df[o] = p.two_f * a;
  if (p.out_dl) p.out_dl[o] = p.f2_dl * g;
}

// RHS slice width: the fewest slices within the register budget (KGP_F64_CAP2 = 28 columns with
// two outputs, 48 with one), each rounded up to a multiple of 4 -- every slice re-evaluates
// the kernel entries, so k = 33 runs as one slice of 36, not 32 + 4
inline int slice_for(int k, int nout, int d) {
  const int cap = nout == 2 ? (d > 8 ? 24 : KGP_F64_CAP2) : 48;  // d > 8: 16 more coordinate registers
  const int nsl = (k + cap - 1) / cap;
  const int w = (k + nsl - 1) / nsl;
  // widths of 2, 18 and 34 are instantiated too (k = 1, 17 and 33: the w-solve, configs[0]'s
  // w + 16 probes and configs[2]'s w + 32 probes), everything else rounds up to a multiple of 4
  if (w <= 2) return 2;
  if (w == 17 || w == 18) return 18;
  if (w == 33 || w == 34) return 34;
  return (w + 3) / 4 * 4;
}

// lane-split dispatch (measured over k = 4..64, d = 2..8, tools/f64_grid.py). Two outputs: k in
// the fewest slices of w <= 64 columns, w = wmin..32 -> 2 lanes x 16, 33..64 -> 4 lanes x {10, 12,
// 14, 16}. One output: only where the one-lane kernel's slice is wmin..36 columns wide (2 x 16 or
// 2 x 18 at the same slice count; four lanes lose to the 40..48-column one-lane slices there).
inline void split_for(int k, int nout, int d, int wmin, int& g, int& kq) {
  g = kq = 0;
  if (nout == 1) {
    const int ks = slice_for(k, 1, d);
    if (ks >= wmin && ks <= 36) {
      g = 2;
      kq = ks <= 32 ? 16 : 18;
    }
    return;
  }
  const int nsl = (k + 63) / 64;
  const int w = (k + nsl - 1) / nsl;
  if (w < wmin) return;
  if (w <= 32) {
    g = 2;
    kq = 16;
    return;
  }
  g = 4;
  kq = ((w + 3) / 4 + 1) / 2 * 2;
  if (kq < 10) kq = 10;
}

using F64Kernel = void (*)(const F64Params);

template <int KT, int NOUT, int DB>
F64Kernel pick_ks(int ks) {
  switch (ks) {
#define KGP_F64_KS(K)                                                                  \
  case K:                                                                              \
    if constexpr (NOUT == 1 || K <= KGP_F64_CAP2) return kmm_f64_kernel<KT, NOUT, K, DB>; \
    [[fallthrough]];
    KGP_F64_KS(2) KGP_F64_KS(4) KGP_F64_KS(8) KGP_F64_KS(12) KGP_F64_KS(16) KGP_F64_KS(18) KGP_F64_KS(20)
    KGP_F64_KS(24) KGP_F64_KS(28) KGP_F64_KS(34)
    KGP_F64_KS(32) KGP_F64_KS(36) KGP_F64_KS(40) KGP_F64_KS(44) KGP_F64_KS(48)
#undef KGP_F64_KS
    default:
      return nullptr;
  }
}

template <int KT, int NOUT, int DB>
F64Kernel pick_split(int g, int kq) {
#define KGP_F64_SPL(GG, KQ) \
  if (g == GG && kq == KQ) return kmm_f64_split_kernel<KT, NOUT, KQ, DB, GG>;
  KGP_F64_SPL(2, 16)
  if constexpr (NOUT == 1) {
    KGP_F64_SPL(2, 18)
  }
  if constexpr (NOUT == 2) {
    KGP_F64_SPL(4, 10) KGP_F64_SPL(4, 12) KGP_F64_SPL(4, 14) KGP_F64_SPL(4, 16)
  }
#undef KGP_F64_SPL
  return nullptr;
}

// the kernel instantiation for (kernel type, outputs, dimension bucket) and either a slice
// width (g = 0) or a lane-split layout (g lanes x kq columns)
template <int KT>
F64Kernel pick_kt(const F64Params& p, int ks, int g, int kq) {
  const bool two = p.out_dl != nullptr;
#define KGP_F64_PICK(NOUT, DB) (g ? pick_split<KT, NOUT, DB>(g, kq) : pick_ks<KT, NOUT, DB>(ks))
  if (p.d <= 4) return two ? KGP_F64_PICK(2, 4) : KGP_F64_PICK(1, 4);
  if (p.d <= 8) return two ? KGP_F64_PICK(2, 8) : KGP_F64_PICK(1, 8);
  return two ? KGP_F64_PICK(2, 16) : KGP_F64_PICK(1, 16);
#undef KGP_F64_PICK
}

// CTAs of `fn` one GPU holds at once (occupancy x SM count), cached per (kernel, device)
int resident_ctas(F64Kernel fn, int threads, int* out) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev = 0;
  KGP_CUDA(cudaGetDevice(&dev));
  const std::pair<const void*, int> key(reinterpret_cast<const void*>(fn), dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return KGP_OK;
    }
  }
  int occ = 0, sms = 0;
  KGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, 0));
  KGP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int w = (occ > 0 ? occ : 1) * (sms > 0 ? sms : 1);
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = w;
  *out = w;
  return KGP_OK;
}

}  // namespace

int launch_kmm_f64(int kt, const F64Params& p_in, DevBuf& ws, cudaStream_t st) {
  KGP_REQUIRE(p_in.d >= 1 && p_in.d <= MAXD, KGP_ERR_INVALID, "fp64 operator supports 1 <= d <= %d, got %d", MAXD,
              p_in.d);
  KGP_REQUIRE(kt >= 0 && kt <= 2, KGP_ERR_INVALID, "unknown kernel id %d", kt);
  if (p_in.nrows <= 0) return KGP_OK;
  F64Params p = p_in;
  // symmetric path: the square operator (rows = columns = all points, the + s B shift on
  // the diagonal), K-type outputs only, k <= 4, n <= 16384 (partials: n / SB x n x k fp64)
  static const bool sym_on = [] {
    const char* e = getenv("KGP_F64_SYM");
    return !(e && atoi(e) == 0);
  }();
  if (sym_on && p.xr == p.xc && p.nrows == p.ncols && p.diag_row0 == 0 && p.out_dl == nullptr && p.k >= 1 &&
      p.k <= 4 && p.ncols <= 16384) {
    const int nb = (int)((p.ncols + SB - 1) / SB);
    int rc = ws.ensure(sizeof(double) * (size_t)nb * p.ncols * p.k);
    if (rc) return rc;
    double* part = ws.as<double>();
    rc = (kt == GAUSS) ? launch_sym<GAUSS>(p, nb, part, st)
                       : (kt == MAT32) ? launch_sym<MAT32>(p, nb, part, st) : launch_sym<MAT52>(p, nb, part, st);
    if (rc) return rc;
    const int64_t cnt = p.ncols * p.k;
    f64_sym_reduce_kernel<<<(unsigned)((cnt + 31) / 32), RW * 32, 0, st>>>(p, nb, part);
    KGP_LAUNCH("f64_sym_reduce_kernel");
    return KGP_OK;
  }
  const int nout = p.out_dl ? 2 : 1;
  // wide RHS blocks: G lanes per row share every kernel-entry evaluation (kmm_f64_split_kernel)
  static const bool split_on = [] {
    const char* e = getenv("KGP_F64_SPLIT");
    return !(e && atoi(e) == 0);
  }();
  // narrowest slice that takes the lane-split kernel, per output count (tools/f64_grid.py)
  static const int wmin1 = [] { const char* e = getenv("KGP_F64_SPLIT_MIN1"); return e ? atoi(e) : 29; }();
  static const int wmin2 = [] { const char* e = getenv("KGP_F64_SPLIT_MIN2"); return e ? atoi(e) : 29; }();
  int sg = 0, skq = 0;
  if (split_on) split_for(p.k, nout, p.d, nout == 2 ? wmin2 : wmin1, sg, skq);
  const int ks = sg ? sg * skq : slice_for(p.k, nout, p.d);
  const int rows_cta = sg ? NTS / sg : NT, threads = sg ? NTS : NT;
  const int64_t rblk = (p.nrows + rows_cta - 1) / rows_cta, kslc = (p.k + ks - 1) / ks;
  const F64Kernel fn = (kt == GAUSS) ? pick_kt<GAUSS>(p, ks, sg, skq)
                                     : (kt == MAT32) ? pick_kt<MAT32>(p, ks, sg, skq) : pick_kt<MAT52>(p, ks, sg, skq);
  KGP_REQUIRE(fn != nullptr, KGP_ERR_INVALID, "fp64 operator slice %d (lanes %d x %d) unsupported", ks, sg, skq);
  // Column split (grid.z): the CTAs run in waves of `wave` = occupancy x SMs, each CTA sweeping
  // ncols / nsplit columns in 64-column tiles, so the time is ~ waves x tiles per CTA. Take the
  // split that minimises that product (the first such; chunks of >= 128 columns): a grid that
  // overflows the last wave by a few CTAs costs a whole extra wave (n = 16384, k = 16, 7 CTAs per
  // SM: 1280 CTAs on 1036 slots ran 2 waves for 1.24 waves of work).
  int wave = 0;
  int rc = resident_ctas(fn, threads, &wave);
  if (rc) return rc;
  static const int nsplit_env = [] {
    const char* e = getenv("KGP_F64_NSPLIT");
    return e ? atoi(e) : 0;
  }();
  const int64_t tiles = (p.ncols + TJ - 1) / TJ;
  int64_t maxsplit = p.ncols / 128 > 0 ? p.ncols / 128 : 1;
  if (maxsplit > 4096) maxsplit = 4096;
  {  // partial sums: at most ~1 GB of workspace
    const int64_t per_split = (int64_t)sizeof(double) * p.nrows * p.k * nout;
    const int64_t cap = ((int64_t)1 << 30) / (per_split > 0 ? per_split : 1);
    if (maxsplit > cap) maxsplit = cap > 1 ? cap : 1;
  }
  int64_t nsplit = 1, best = -1;
  for (int64_t ns = 1; ns <= maxsplit; ++ns) {
    const int64_t ctas = rblk * kslc * ns;
    const int64_t waves = (ctas + wave - 1) / wave;
    const int64_t per = (tiles + ns - 1) / ns;  // tiles per CTA
    // one extra tile-equivalent per CTA for its prologue / epilogue and partial-sum traffic
    const int64_t cost = waves * (per + 1);
    if (best < 0 || cost < best) {
      best = cost;
      nsplit = ns;
    }
    if (ctas >= 64 * (int64_t)wave) break;  // many waves: the tail no longer matters
  }
  if (nsplit_env > 0) nsplit = nsplit_env < maxsplit ? nsplit_env : maxsplit;
  p.jchunk = ((p.ncols + nsplit - 1) / nsplit + TJ - 1) / TJ * TJ;
  nsplit = (p.ncols + p.jchunk - 1) / p.jchunk;
  p.part = nullptr;
  p.part_stride = 0;
  if (nsplit > 1) {
    const int64_t per = nsplit * p.nrows * p.k;
    rc = ws.ensure(sizeof(double) * per * (p.out_dl ? 2 : 1));
    if (rc) return rc;
    p.part = ws.as<double>();
    p.part_stride = per;
  }
  dim3 grid((unsigned)rblk, (unsigned)kslc, (unsigned)nsplit);
  fn<<<grid, threads, 0, st>>>(p);
  KGP_LAUNCH(sg ? "kmm_f64_split_kernel" : "kmm_f64_kernel");
  if (nsplit == 1) return KGP_OK;
  const int64_t cnt = p.nrows * p.k;
  f64_reduce_kernel<<<(unsigned)((cnt + 31) / 32), RW * 32, 0, st>>>(p, (int)nsplit);
  KGP_LAUNCH("f64_reduce_kernel");
  return KGP_OK;
}

}  // namespace kgp
