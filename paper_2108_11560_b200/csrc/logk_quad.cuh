// logk_quad.cuh -- fixed-bin trapezoid quadrature in log-sum-exp form
// (PAPER.md Eq. (int)) with the derivative integrands of Sec. 4.1
// accumulated in the same pass over f's nodes (R14).
//
// With shift s ~ g(t_p) and q = e^{-2vt}:
//   exp(g(t) - s)                 = E (1 + q),   E = exp(vt - x cosh t - s - log 2)
//   t tanh(vt) exp(g(t) - s)      = E t (1 - q)
//   cosh t exp(g(t) - s)          = E (1 + q) cosh t
// so one exponential per node carries all three sums.
//
// Node loops:
//   nodes_fp64_v2  the default FP64 loop: every FP64 instruction reads at most
//                  two 64-bit registers (B200 register-file banks), x folded
//                  into the cosh recurrence, E (1 - q) = 2E - w, exact-start
//                  group-step recurrences (no re-anchoring);
//   nodes_fp64     the general loop: p = 1 - q by an additive recurrence (no
//                  cancellation for small vt, R21), e^{+-t} re-anchored every
//                  kAnchor nodes, exp clamp for ranges far below eps;
//   quad_f32_v3    FP32 entry point: one FP64 fixed-point exponent per 4
//                  nodes, FP32 offsets and f32x2 node pairs, MUFU.EX2;
//                  quad_f32 its fallback for ranges far below eps.
// The half weights of the two end nodes are taken back outside
// the loops, so the loop bodies carry no per-node select.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "logk_range.cuh"

namespace blk {

constexpr int kExpBits = 11;
constexpr int kExpTab = 1 << kExpBits;   // 2^(j/2048), j = 0..2047, in shared memory (16 KB)
#ifndef BLK_ANCHOR
#define BLK_ANCHOR 44
#endif
constexpr int kAnchor = BLK_ANCHOR; // v1 loop: FP64 re-anchoring interval for e^{+-t} (nodes)
#ifndef BLK_GROUP
#define BLK_GROUP 4
#endif
#ifndef BLK_MINB
// __launch_bounds__ min blocks per SM: 4 (112 registers, 16 warps/SM).  The v2
// loop with each group's cosh factors formed from the group base (BLK_X_DIRECT)
// needs the room: at 5 blocks (<= 102 registers) ptxas re-schedules it to 102
// instructions (-5%), at 4 it is 94 instructions with 167 operand-read cycles
// per 4 nodes instead of 97 / 174: c3 +2.9%, c5 +2.7%, c2 +2.3%
// (profiles/r02zzg_xdirect*.log).  (Round 1: 6 capped it at 78 registers and
// cost 2-2.5%; without BLK_X_DIRECT 4 and 5 measure the same.)
#define BLK_MINB 4
#endif
constexpr int kGroup = BLK_GROUP; // nodes evaluated together (independent exp chains)
#ifndef BLK_GROUP2
#define BLK_GROUP2 4
#endif
constexpr int kGroup2 = BLK_GROUP2; // v2 loop group size
#ifndef BLK_V2_UNROLL
#define BLK_V2_UNROLL 1
#endif
constexpr int kV2Unroll = BLK_V2_UNROLL; // tuning knob: unroll of the v2 group loop
#ifndef BLK_X_DIRECT
// v2 loop: X_j = x cosh t_j of the group's nodes j = 1..3 as Xp_c e^{jh} + Xm_c
// e^{-jh} from the group base (one FMUL + one FMA, no chain through the group)
// instead of the Xp, Xm recurrences plus a sum: 3 FP64 instructions and 7
// operand-read cycles fewer per group (BLK_MINB)
#define BLK_X_DIRECT 1
#endif
#ifndef BLK_S1_SPLIT
#define BLK_S1_SPLIT 1
#endif
constexpr bool kS1Split = BLK_S1_SPLIT;   // v2 loop: S1 as t_c sum Ep + h sum j Ep per group

// 2^(j/2048) with (j << 9) subtracted from the high word (gen_exp2_table.py):
// adding (k << 9) to the high word of entry k & 2047 gives 2^(k/2048) for
// any k in [-2^21, 2^21) -- the 2^(k >> 11) scale costs one integer
// multiply-add and no shift.
__device__ __align__(16) const unsigned long long kExp2TablePc[kExpTab] = {
#include "exp2_table_pc.inc"
};

// The shared-memory copy of the table, one per CTA of every kernel that
// uses exp_tab.  A file-scope __shared__ array lets LDS address it with an
// immediate/uniform base (no per-node base-register add).
__shared__ __align__(16) double g_exp_tab[kExpTab];

#ifndef BLK_TMA_TABLE
#define BLK_TMA_TABLE 1
#endif
// The table copy to shared memory, complete and visible to the whole block on
// return.  BLK_TMA_TABLE: one bulk asynchronous copy (TMA engine,
// cp.async.bulk global -> shared, 16 KB) issued by thread 0 and signalled
// through an mbarrier transaction count, instead of every thread moving its
// share through registers (8 LDG.128 + 8 STS.128 per thread of a 128-thread
// block).
__shared__ __align__(8) unsigned long long g_tab_bar;
__device__ __forceinline__ void load_exp_table_sync() {
#if BLK_TMA_TABLE
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&g_tab_bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(g_exp_tab);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((unsigned)sizeof(g_exp_tab)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(kExp2TablePc), "r"((unsigned)sizeof(g_exp_tab)), "r"(bar)
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar) : "memory");
#else
  const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(kExp2TablePc);
  ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(g_exp_tab);
  for (int j = threadIdx.x; j < kExpTab / 2; j += blockDim.x) dst[j] = src[j];
  __syncthreads();
#endif
}

// 2^(k/2048) for k in [-2^21, 2^21): one LDS.64 and one IMAD.
__device__ __forceinline__ double exp_scale(int k) {
  // explicit 32-bit shared address (and, shl, add -> LOP3 + LEA): left to
  // itself ptxas folds the table base into the LDS only while it can keep it
  // in a uniform register, and loses that with any per-lane branch ahead of
  // the node loop (one extra integer add per node)
  const unsigned base = (unsigned)__cvta_generic_to_shared(g_exp_tab);
  unsigned addr;
  asm("{\n\t.reg .u32 t;\n\tand.b32 t, %1, 2047;\n\tshl.b32 t, t, 3;\n\tadd.u32 %0, t, %2;\n\t}"
      : "=r"(addr) : "r"(k), "r"(base));
  // volatile: the compiler must not move the read above the barrier that
  // follows load_exp_table (a plain asm is free to move, it has no memory
  // dependence)
  double tj;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(tj) : "r"(addr));
  return __hiloint2double(k * 512 + __double2hiint(tj), __double2loint(tj));
}

constexpr double kExpInvL = 2954.639443740597;       // 2048 / ln 2
constexpr double kExpMagic = 6755399441055744.0;     // 1.5 * 2^52: round-to-int trick
constexpr double kExpC = 0.0003384507717577858;      // ln2/2048 (single-step reduction:
                                                     // |k| <= 2.1e6 -> |error| < 6e-14 |a|/707)
constexpr double kExpClo = 1.1323470770733885e-20;   // ln2/2048 - kExpC
// -ln2/2048 as a constant-bank operand for the node loops: fma(kd, -C, a)
// with C in a general register reads three distinct 64-bit registers (one
// extra issue cycle); ptxas keeps a __constant__ operand in the
// constant bank (it otherwise picks a uniform or a general register depending
// on what else the kernel holds).
__constant__ double kNegExpCc = -0.0003384507717577858;

// e^r - 1 for |r| <= ln2/4096 (truncation r^4/24 < 3.5e-17): Horner, every
// operation with at most two register operands (the FP64 pipe issues an
// instruction reading three distinct 64-bit registers in 3 cycles, not 2:
// two register-file banks).
__device__ __forceinline__ double exp_em1(double r) {
  double p = fma(r, 1.6666666666666666e-01, 0.5);
  p = fma(p, r, 1.0);
  return p * r;
}

// exp(a) by Tang's table method: a = (k/2048) ln2 + r, |r| <= ln2/4096,
// exp(a) = 2^(k/2048) * (1 + em1(r)).  Valid for a in [-707, 709]; CLAMP maps
// a < -707 to e^-707 (caller decides whether its arguments can leave the
// range -- see quad_f64).  7 FP64-pipe instructions + LDS.64 + 3 integer ops.
template <bool CLAMP>
__device__ __forceinline__ double exp_tab(double a) {
  if (CLAMP) a = a < -707.0 ? -707.0 : a;
  double kd = fma(a, kExpInvL, kExpMagic);
  const int k = __double2loint(kd);
  kd -= kExpMagic;
  const double r = fma(kd, -kExpC, a);
  const double ts = exp_scale(k);
  return fma(ts, exp_em1(r), ts);
}
template <bool CLAMP>
__device__ __forceinline__ double exp_tab(double a, const double *) { return exp_tab<CLAMP>(a); }

// 1/a to ~1 ulp: MUFU.RCP64H seed + two Newton steps.
__device__ __forceinline__ double rcp64(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

// e^h - 1 for 0 <= h < ln 2 to ~1 ulp of the result (once per lane, for
// the cosh recurrence steps of the v2 loop): e^{h/2} - 1 by its Taylor
// series to degree 13 (all terms positive; truncation < 2e-17 relative for
// h/2 <= 0.35), then e^h - 1 = u (u + 2).
__device__ __forceinline__ double expm1_small(double h) {
  const double y = 0.5 * h;
  double p = fma(y, 1.0 / 6227020800.0, 1.0 / 479001600.0);   // 1/13!, 1/12!
  p = fma(p, y, 1.0 / 39916800.0);
  p = fma(p, y, 1.0 / 3628800.0);
  p = fma(p, y, 1.0 / 362880.0);
  p = fma(p, y, 1.0 / 40320.0);
  p = fma(p, y, 1.0 / 5040.0);
  p = fma(p, y, 1.0 / 720.0);
  p = fma(p, y, 1.0 / 120.0);
  p = fma(p, y, 1.0 / 24.0);
  p = fma(p, y, 1.0 / 6.0);
  p = fma(p, y, 0.5);
  p = fma(p, y, 1.0);
  const double u = p * y;
  return fma(u, u, 2.0 * u);
}

// log(y) for normal positive y with the exp table (the epilogue's
// log(h S0)): y = 2^e m, m in [1, 2); k = round(2048 log2 m) from MUFU.LG2,
// m 2^{-k/2048} = 1 + r with |r| < 2^-11 (the table entry for -k), log1p(r)
// by its series to r^5 (truncation < 1e-19 relative), and (2048 e + k) ln2/2048
// with a two-part constant.  ~2 ulp of the table entry and the product: an
// absolute error < 3e-16, against ~29 FP64 instructions for libdevice log.
__device__ __forceinline__ double log_tab(double y) {
  const int hi = __double2hiint(y);
  const int e = (hi >> 20) - 1023;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(y));
  float l2;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(__double2float_rn(m)));
  const int k = __float2int_rn(l2 * 2048.0f);            // 0 .. 2048
  const double r = m * exp_scale(-k) - 1.0;
  double p = fma(r, 0.2, -0.25);
  p = fma(p, r, 1.0 / 3.0);
  p = fma(p, r, -0.5);
  const double l1 = fma(p * r, r, r);
  const double kk = (double)(e * 2048 + k);
  return fma(kk, kExpC, fma(kk, kExpClo, l1));
}

// log(y) of the epilogue's y = h S0: log_tab on normal finite y, libm for the
// rest (0, subnormal, inf: not reached by valid ranges).
__device__ __forceinline__ double log_sum(double y) {
  return (y >= 2.2250738585072014e-308 && y < 1.7e308) ? log_tab(y) : log(y);
}

// 1 - e^z for z <= 0 without cancellation (-expm1(z)).
__device__ __forceinline__ double one_minus_exp(double z) {
  if (z < -0.34657359027997264) return 1.0 - exp_tab<true>(z);
  // Taylor series of -(e^z - 1) to z^14 (|z| <= ln2/2: truncation < 3e-18 |z|)
  double p = 1.0 / 87178291200.0;   // 1/14!
  p = fma(p, z, 1.0 / 6227020800.0);
  p = fma(p, z, 1.0 / 479001600.0);
  p = fma(p, z, 1.0 / 39916800.0);
  p = fma(p, z, 1.0 / 3628800.0);
  p = fma(p, z, 1.0 / 362880.0);
  p = fma(p, z, 1.0 / 40320.0);
  p = fma(p, z, 1.0 / 5040.0);
  p = fma(p, z, 1.0 / 720.0);
  p = fma(p, z, 1.0 / 120.0);
  p = fma(p, z, 1.0 / 24.0);
  p = fma(p, z, 1.0 / 6.0);
  p = fma(p, z, 0.5);
  p = fma(p, z, 1.0);
  return -(p * z);
}

// exp(a), a in [-707, 709.78], with a two-part (Cody-Waite) ln2/2048 (no
// reduction error: ~0.5 ulp from the table entry plus the final rounding);
// for the FP64 range finder.  Its constants differ from exp_tab's on
// purpose: sharing them with this rarely taken path, ptxas moved the node
// loops' reduction constant to a general register (a three-register DFMA in
// every node).
__device__ __forceinline__ double exp_cw(double a) {
  double kd = fma(a, kExpInvL, kExpMagic);
  const int k = __double2loint(kd);
  kd -= kExpMagic;
  double r = fma(kd, -3.384507715509244e-04, a);   // hi part: 31-bit mantissa, kd * hi exact
  r = fma(kd, -2.0686139481490644e-13, r);
  const double ts = exp_scale(k);
  return fma(ts, exp_em1(r), ts);
}

#ifndef BLK_PLAN_LOG_TAB
#define BLK_PLAN_LOG_TAB 1
#endif
// FP64 range-finder point evaluations with the table exp and rcp64 instead
// of libdevice exp and IEEE division (kernels that load the exp table):
// 3-4x fewer instructions per evaluation, ~1 ulp like the libm calls.
struct PlanF64Tab {
  double v, x, hx, v2, m2v;
  // e^{+-t}, overflowing to (inf, 0) past 709.78 like libm (FindRange's far
  // probes: F = -inf there, as in the oracle)
  __device__ __forceinline__ void ep(double t, double &e, double &ei) const {
    const bool fin = t < 709.78;
    e = exp_cw(fmin(t, 709.78));
    ei = rcp64(e);
    if (!fin) { e = __longlong_as_double(0x7ff0000000000000ULL); ei = 0.0; }
  }
  __device__ __forceinline__ void parts(double t, double &e, double &ei, double &q, double &r) const {
    ep(t, e, ei);
    q = exp_cw(fmax(m2v * t, -707.0));
    r = rcp64(1.0 + q);
  }
  __device__ __forceinline__ void peak(double t, double &F, double &dF) const {
    double e, ei, q, r;
    parts(t, e, ei, q, r);
    F = v * ((1.0 - q) * r) - hx * (e - ei);
    dF = v2 * (4.0 * q * r * r) - hx * (e + ei);
  }
  __device__ __forceinline__ void thr(double c, double t, double &F, double &dF) const {
    double e, ei, q, r;
    parts(t, e, ei, q, r);
    F = v * t + log1p_q(q) - hx * (e + ei) - c;
    dF = v * ((1.0 - q) * r) - hx * (e - ei);
  }
  __device__ __forceinline__ double gval(double t) const {
    double e, ei;
    ep(t, e, ei);
    return v * t + log1p_q(exp_cw(fmax(m2v * t, -707.0))) - kLn2 - hx * (e + ei);
  }
  // log(1 + q) for q = e^{-2vt} in [0, 1]: the table log of 1 + q, absolute
  // error < 4e-16 (the rounding of 1 + q included) -- F's other terms carry
  // at least that much -- against ~30 instructions of libdevice log1p
  __device__ __forceinline__ static double log1p_q(double q) {
#if BLK_PLAN_LOG_TAB
    return log_tab(1.0 + q);
#else
    return log1p(q);
#endif
  }
};
__device__ __forceinline__ Plan<double> make_plan_f64_tab(double v, double x, double log_eps) {
  return make_plan_f64_with(PlanF64Tab{v, x, 0.5 * x, v * v, -2.0 * v}, v, x, log_eps);
}

struct Sums64 {
  double S0, S1, S2;        // sum w, sum E t p, sum w cosh t      (Sec. 4.1, first order)
  double S11, S22, S12;     // sum w t^2, sum w cosh^2 t, sum E t p cosh t (second order)
};

// Accumulates one node: E = exp(vt - x cosh t - s - log 2), q = e^{-2vt},
// p = 1 - q, so w = E (1 + q) = e^{g(t) - s} and E t p = t tanh(vt) e^{g - s}.
template <bool DV, bool DX, bool HESS>
__device__ __forceinline__ void accumulate(Sums64 &s, double E, double q, double p, double t,
                                           double ch) {
  const double w = fma(E, q, E);
  s.S0 += w;
  if (HESS) {
    const double wc = w * ch, wt = w * t, etp = (E * t) * p;
    s.S2 += wc;
    s.S22 = fma(wc, ch, s.S22);
    s.S11 = fma(wt, t, s.S11);
    s.S1 += etp;
    s.S12 = fma(etp, ch, s.S12);
  } else {
    if (DX) s.S2 = fma(w, ch, s.S2);
    if (DV) s.S1 = fma(E * t, p, s.S1);
  }
}

// One node's contributions, given cosh t, q and p.
template <bool DV, bool DX, bool HESS, bool CLAMP>
__device__ __forceinline__ void node_acc(double v, double x, double s_mid, double t, double ch,
                                         double q, double p, Sums64 &s) {
  accumulate<DV, DX, HESS>(s, exp_tab<CLAMP>(fma(-x, ch, fma(v, t, -s_mid))), q, p, t, ch);
}

// v1 node loop (general): nodes [ib, ie) with weight 1.  Node positions are
// t0 + m h to 1 ulp (an accumulated t += h would drift by m ulp, which v t
// amplifies for large v); e^{+-t} are re-anchored every kAnchor nodes, q and
// p advance across chunks; p = 1 - q by an additive recurrence (no
// cancellation for small v t, R21).  Used for the second-order sums, for
// 0 < v < 1e-5 and for ranges that need the exp clamp.
template <bool DV, bool DX, bool HESS, bool CLAMP>
__device__ __forceinline__ void nodes_fp64(double v, double x, double t0, double h,
                                           double s_mid, int ib, int ie, Sums64 &out) {
  if (ie <= ib) return;
  constexpr bool NEEDP = DV || HESS;
  const double m2v = -2.0 * v;
  const double eh = exp_tab<false>(h);
  const double ehi = rcp64(eh);
  const double tb = fma((double)ib, h, t0);
  double q = exp_tab<true>(m2v * tb);           // q_m = e^{-2 v t_m}
  const double eq = exp_tab<true>(m2v * h);
  double p = NEEDP ? one_minus_exp(m2v * tb) : 0.0;  // p_m = 1 - q_m
  const double a1 = NEEDP ? one_minus_exp(m2v * h) : 0.0;
  Sums64 s{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  static_assert(kAnchor % kGroup == 0, "anchor interval must hold whole groups");
#pragma unroll 1
  for (int c0 = ib; c0 < ie; c0 += kAnchor) {
    const int c1 = min(c0 + kAnchor, ie);
    double tc = fma((double)c0, h, t0);
    double et = 0.5 * exp_tab<true>(fmin(tc, 709.0));   // e^t / 2
    double eti = 0.25 * rcp64(et);                       // e^-t / 2
    if (c0 == 0) {
      // node 0 has weight 1/2: take half of it back.  It is exact
      // here (anchored state) and may be the largest node (t0 = 0 when the
      // peak region reaches t = 0), so this correction is done in FP64.
      Sums64 z{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      node_acc<DV, DX, HESS, CLAMP>(v, x, s_mid, tc, et + eti, q, p, z);
      s.S0 -= 0.5 * z.S0; s.S1 -= 0.5 * z.S1; s.S2 -= 0.5 * z.S2;
      s.S11 -= 0.5 * z.S11; s.S22 -= 0.5 * z.S22; s.S12 -= 0.5 * z.S12;
    }
    int m = c0;
#pragma unroll 1
    for (; m + kGroup <= c1; m += kGroup) {          // groups of kGroup nodes
      double tg[kGroup], chg[kGroup], qg[kGroup], pg[kGroup];
#pragma unroll
      for (int j = 0; j < kGroup; ++j) {
        tg[j] = j == 0 ? tc : fma(double(j), h, tc);
        chg[j] = et + eti;
        et *= eh;
        eti *= ehi;
        qg[j] = q;
        pg[j] = p;
        if (NEEDP) p = fma(q, a1, p);
        q *= eq;
      }
      // the group's exponentials stage by stage, so consecutive dependent
      // FP64 instructions of one node are kGroup instructions apart
      double a[kGroup], kd[kGroup], r[kGroup], ts[kGroup];
      int k[kGroup];
#pragma unroll
      for (int j = 0; j < kGroup; ++j) a[j] = fma(v, tg[j], -s_mid);
#pragma unroll
      for (int j = 0; j < kGroup; ++j) {
        a[j] = fma(-x, chg[j], a[j]);
        if (CLAMP) a[j] = a[j] < -707.0 ? -707.0 : a[j];
      }
#pragma unroll
      for (int j = 0; j < kGroup; ++j) kd[j] = fma(a[j], kExpInvL, kExpMagic);
#pragma unroll
      for (int j = 0; j < kGroup; ++j) {
        k[j] = __double2loint(kd[j]);
        kd[j] -= kExpMagic;
      }
#pragma unroll
      for (int j = 0; j < kGroup; ++j) ts[j] = exp_scale(k[j]);
#pragma unroll
      for (int j = 0; j < kGroup; ++j) r[j] = fma(kd[j], kNegExpCc, a[j]);
#pragma unroll
      for (int j = 0; j < kGroup; ++j) {
        const double E = fma(ts[j], exp_em1(r[j]), ts[j]);
        accumulate<DV, DX, HESS>(s, E, qg[j], pg[j], tg[j], chg[j]);
      }
      tc = fma((double)(m + kGroup), h, t0);
    }
#pragma unroll 1
    for (; m < c1; ++m) {                            // remainder
      node_acc<DV, DX, HESS, CLAMP>(v, x, s_mid, tc, et + eti, q, p, s);
      if (NEEDP) p = fma(q, a1, p);
      q *= eq;
      et *= eh; eti *= ehi;
      tc = fma((double)(m + 1), h, t0);
    }
  }
  out.S0 += s.S0; out.S1 += s.S1; out.S2 += s.S2;
  out.S11 += s.S11; out.S22 += s.S22; out.S12 += s.S12;
}

// v2 node loop (first-order sums, no exp clamp, v = 0 or v >= 1e-5):
// the same nodes and sums, arranged so that almost every FP64 instruction
// reads at most two distinct 64-bit registers (a third costs
// a full extra issue cycle on B200):
//   * x is folded into the cosh recurrence: X = x cosh t = Xp + Xm with
//     Xp = (x/2) e^t, Xm = (x/2) e^{-t}; S2 is accumulated as sum w X and
//     divided by x once at the end;
//   * v t - s = B_j = B_c + j (v h) from the group base B_c = v t_c - s
//     (immediate j), so the exponent is a = B_j - X_j;
//   * E t p = E (1 - q) t with E (1 - q) = 2E - w (w = E (1 + q)): the
//     rounding of w costs ~eps/(2 v t_w) of S1 (t_w the weighted mean node
//     position, >= t1/2 here), so the caller takes this loop only when
//     v t1 >= 1e-3 (error < 3e-13) or v = 0 (exactly 0); smaller v t1 takes
//     the v1 loop;
//   * e^{+-t} and q advance per group by e^{+-G h}, e^{-2 v G h} and inside
//     the group by e^{+-h}, e^{-2 v h}, no re-anchoring.  The group steps
//     of the cosh factors are X <- X + X u with u = e^{+-Gh} - 1 from an
//     accurate expm1: a rounded multiplier e^{+-Gh} would add the same
//     relative error at every step, a systematic drift of (n/G) ulp of X in
//     the exponent -- 2e-11 absolute where x cosh t ~ 1e4 cancels against
//     v t to a small g (test_large_order_cancellation); with u it is ~|u|
//     ulp per step.  Same instruction count (an FMA reading two distinct
//     registers instead of a DMUL).
// One node of the v2 loop: E = e^{a}, w = E (1 + q), Ep = 2E - w = E (1 - q)
// (S1 term / t), X = x cosh t.  HESS adds the second-order sums in the
// scaled form S22x = sum w X^2 = x^2 S22 and S12x = sum Ep t X = x S12.
template <bool DV, bool DX, bool HESS>
__device__ __forceinline__ void v2_accumulate(double E, double q, double X, double t, double &S0,
                                              double &S1, double &S2, double &S11, double &S22,
                                              double &S12) {
  const double w = fma(E, q, E);
  S0 += w;
  if (HESS) {
    const double wX = w * X, wt = w * t, ept = fma(E, 2.0, -w) * t;
    S2 += wX;
    S22 = fma(wX, X, S22);
    S11 = fma(wt, t, S11);
    S1 += ept;
    S12 = fma(ept, X, S12);
  } else {
    if (DX) S2 = fma(w, X, S2);
    if (DV) S1 = fma(fma(E, 2.0, -w), t, S1);
  }
}

#ifndef BLK_HALF_IN_REM
#define BLK_HALF_IN_REM 1
#endif
// half_last: node ie - 1 is node n (this lane owns it); when it falls in the
// remainder loop (the node count is not a multiple of G, e.g. n = 128) it is
// taken there with its trapezoid weight 1/2 and the function returns
// true -- no separate end-node correction needed.
template <bool DV, bool DX, bool HESS = false>
__device__ __forceinline__ bool nodes_fp64_v2(double v, double x, double t0, double h,
                                              double s_mid, int ib, int ie, Sums64 &out,
                                              bool half_last = false) {
  if (ie <= ib) return false;
  constexpr int G = kGroup2;
  const double m2v = -2.0 * v, vh = v * h;
  const double tb = fma((double)ib, h, t0);
  const double eb = exp_tab<true>(fmin(tb, 709.0));
  const double hx = 0.5 * x;
  double XpG = hx * eb, XmG = hx * rcp64(eb);
  static_assert(G == 4, "uG below is (1 + u1)^4 - 1");
  // e^{+-h} - 1 and e^{+-Gh} - 1 for the steps X <- X + X u (u1 to ~1 ulp
  // for h < ln 2; beyond, e^h - 1 is no more precise than e^h itself).
  // Branch-free: the lanes of a warp would take both sides.  Capped like the
  // exp arguments at 709: only ranges reaching e^t ~ 1e308 (x < 1e-300) get
  // there, where those nodes underflow either way.
  const double u1c = exp_tab<false>(fmin(h, 709.0)) - 1.0, u1a = expm1_small(h);
  const double u1 = fmin(h < 0.6931 ? u1a : u1c, 8e307);
  const double uG = fmin(u1 * fma(u1, fma(u1, 4.0 + u1, 6.0), 4.0), 8e307);  // e^{Gh} - 1
  const double u1i = -u1 * rcp64(1.0 + u1);                                  // e^{-h} - 1
  const double uGi = u1i * fma(u1i, fma(u1i, 4.0 + u1i, 6.0), 4.0);          // e^{-Gh} - 1
  double qG = exp_tab<true>(m2v * tb);
  const double eq1 = exp_tab<true>(m2v * h);
  // e^{-2v G h} by squaring: q only enters w = E (1 + q), where a few ulp of
  // drift over n/G steps are far below the other rounding (measured +1%)
  const double eq2 = eq1 * eq1, eqG = eq2 * eq2;
#if BLK_X_DIRECT
  // e^{+-jh}, j = 1..3: X_j = Xp_c e^{jh} + Xm_c e^{-jh} from the group base
  // (one rounding each, no chain inside the group)
  // (capped like u1: a coarse grid's e^{2h} may pass DBL_MAX; 0 * inf must not
  // turn an underflowed X+ into NaN)
  const double ej1 = 1.0 + u1, ej2 = fmin(ej1 * ej1, 8e307), ej3 = fmin(ej2 * ej1, 8e307);
  const double ei1 = 1.0 + u1i, ei2 = ei1 * ei1, ei3 = ei2 * ei1;
#endif
  double S0 = 0.0, S1 = 0.0, S2 = 0.0, S11 = 0.0, S22 = 0.0, S12 = 0.0, S1j = 0.0;
  if (ib == 0) {
    // node 0 carries weight 1/2: take half of it back (exact state)
    const double X = XpG + XmG;
    const double E = exp_tab<false>(fma(v, t0, -s_mid) - X);
    v2_accumulate<DV, DX, HESS>(-0.5 * E, qG, X, t0, S0, S1, S2, S11, S22, S12);
  }
  double md = (double)ib;
  int m = ib;
#pragma unroll (kV2Unroll)
  for (; m + G <= ie; m += G) {
    const double tc = fma(md, h, t0);
    md += (double)G;
    const double Bc = fma(v, tc, -s_mid);
    double X[G], a[G], q[G], kd[G], r[G], ts[G];
    int k[G];
#if BLK_X_DIRECT
    double qq = qG;
    X[0] = XpG + XmG;
    X[1] = fma(XpG, ej1, XmG * ei1);
    X[2] = fma(XpG, ej2, XmG * ei2);
    X[3] = fma(XpG, ej3, XmG * ei3);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      q[j] = qq;
      if (j + 1 < G) qq *= eq1;
    }
#else
    double xp = XpG, xm = XmG, qq = qG;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      X[j] = xp + xm;
      q[j] = qq;
      if (j + 1 < G) { xp = fma(xp, u1, xp); xm = fma(xm, u1i, xm); qq *= eq1; }
    }
#endif
    XpG = fma(XpG, uG, XpG); XmG = fma(XmG, uGi, XmG); qG *= eqG;
#pragma unroll
    for (int j = 0; j < G; ++j) a[j] = (j == 0 ? Bc : fma(double(j), vh, Bc)) - X[j];
#pragma unroll
    for (int j = 0; j < G; ++j) kd[j] = fma(a[j], kExpInvL, kExpMagic);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      k[j] = __double2loint(kd[j]);
      kd[j] -= kExpMagic;
    }
#pragma unroll
    for (int j = 0; j < G; ++j) ts[j] = exp_scale(k[j]);
#pragma unroll
    for (int j = 0; j < G; ++j) r[j] = fma(kd[j], kNegExpCc, a[j]);
    if (HESS || !DV || !kS1Split) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const double E = fma(ts[j], exp_em1(r[j]), ts[j]);
        v2_accumulate<DV, DX, HESS>(E, q[j], X[j], j == 0 ? tc : fma(double(j), h, tc), S0,
                                    S1, S2, S11, S22, S12);
      }
    } else {
      // S1 = sum Ep_j (t_c + j h) = t_c sum Ep_j + h sum j Ep_j: per group one
      // three-register FMA instead of four (Ep = E (1 - q) >= 0, no cancellation)
      double Ep[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const double E = fma(ts[j], exp_em1(r[j]), ts[j]);
        const double w = fma(E, q[j], E);
        S0 += w;
        if (DX) S2 = fma(w, X[j], S2);
        Ep[j] = fma(E, 2.0, -w);
      }
      static_assert(G == 4, "S1 split below is written for groups of 4");
      const double A = (Ep[0] + Ep[1]) + (Ep[2] + Ep[3]);
      S1 = fma(tc, A, S1);
      S1j += fma(Ep[3], 3.0, fma(Ep[2], 2.0, Ep[1]));
    }
  }
  double xp = XpG, xm = XmG, qq = qG;
  const double tr = fma(md, h, t0);
  const bool half_rem = BLK_HALF_IN_REM && half_last && m < ie;
#pragma unroll 1
  for (; m < ie; ++m) {                             // remainder, one node at a time
    const double t = fma((double)m - md, h, tr);
    const double X = xp + xm;
    double E = exp_tab<false>(fma(v, t, -s_mid) - X);
    if (half_rem && m == ie - 1) E *= 0.5;           // node n: weight 1/2
    v2_accumulate<DV, DX, HESS>(E, qq, X, t, S0, S1, S2, S11, S22, S12);
    xp = fma(xp, u1, xp); xm = fma(xm, u1i, xm); qq *= eq1;
  }
  const double rx = rcp64(x);
  out.S0 += S0;
  if (DV || HESS) out.S1 += fma(h, S1j, S1);
  if (DX || HESS) out.S2 += S2 * rx;
  if (HESS) {
    out.S11 += S11;
    out.S22 += (S22 * rx) * rx;
    out.S12 += S12 * rx;
  }
  return half_rem;
}

// Half of the last node's contributions, evaluated in FP32: that node sits
// below the eps level of the peak (d(t1) < 0), so its terms are < 2^-52 of
// the sums and FP32 is exact to far below double rounding there.
template <bool DV, bool DX, bool HESS>
__device__ __forceinline__ void end_half_f32(double v, double x, double s_mid, double t,
                                             Sums64 &s) {
  const float kL2e = 1.4426950408889634f;
  const float tf = float(t), vf = float(v);
  const float e = ex2_approx(tf * kL2e);
  const float ch = 0.5f * (e + rcp_approx(e));
  const float q = ex2_approx(-2.0f * vf * kL2e * tf);
  const float arg = float(fma(v, t, -s_mid) - x * double(ch));
  const float E = 0.5f * ex2_approx(arg * kL2e);
  const float w = fmaf(E, q, E);
  if (!(w > 0.0f)) return;          // underflowed (or e^t overflowed FP32): nothing to take back
  const double etp = double(E * tf) * (-expm1f(-2.0f * vf * tf));
  s.S0 -= w;
  if (DX || HESS) s.S2 -= double(w) * ch;
  if (DV || HESS) s.S1 -= etp;
  if (HESS) {
    s.S11 -= double(w) * tf * tf;
    s.S22 -= double(w) * ch * ch;
    s.S12 -= etp * ch;
  }
}

// The same in FP64 (exact state, libm-accurate cosh, clamped exponent): for
// coarse grids (n < kEndF32MinBins), whose sums can miss the peak by far more
// than the node's own eps level -- at 2 bins over a range 30 wide the sums
// are of the same order as node n's term.
template <bool DV, bool DX, bool HESS>
__device__ __forceinline__ void end_half_f64(double v, double x, double s_mid, double t,
                                             Sums64 &s) {
  const double et = exp_cw(fmin(t, 709.0));
  const double ch = 0.5 * (et + rcp64(et));
  const double z2 = fmax(-2.0 * v * t, -707.0);
  Sums64 z{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  node_acc<DV, DX, HESS, true>(v, x, s_mid, t, ch, exp_cw(z2), one_minus_exp(z2), z);
  s.S0 -= 0.5 * z.S0; s.S1 -= 0.5 * z.S1; s.S2 -= 0.5 * z.S2;
  s.S11 -= 0.5 * z.S11; s.S22 -= 0.5 * z.S22; s.S12 -= 0.5 * z.S12;
}
// From this many bins the node nearest the peak is within 36/n^2 < 0.01 (log
// units) of it, so S0 is at least ~the peak term and node n's (< eps of the
// peak) is resolved by FP32 (FP64 quadrature) or below FP32 resolution
// altogether (FP32 quadrature, which leaves it out).
constexpr int kEndF32MinBins = 64;

// Nodes [mb, me) of the n-interval trapezoid on [t0, t0 + n h] (node m at
// t0 + m h; nodes 0 and n carry weight 1/2: all nodes are summed
// with weight 1 and half of each end node is taken back).  The lane owning
// node 0 has mb == 0, the lane owning node n has mb < me == n + 1 (lanes past
// the last node get the empty range mb == me == n + 1 and take nothing back).
template <bool DV, bool DX, bool CLAMP, bool HESS = false>
__device__ __forceinline__ Sums64 quad_f64(double v, double x, double t0, double h,
                                           double shift, int n, int mb, int me,
                                           const double *__restrict__ tab) {
  Sums64 s{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const double s_mid = shift + kLn2;                 // E = exp(vt - x cosh t - s_mid)
  (void)tab;
  const bool own_n = mb < me && me == n + 1;
  bool n_done = false;
#ifndef BLK_QUAD_V1
  if (!CLAMP && !(v > 0.0 && v * fma((double)n, h, t0) < 1e-3))
    n_done = nodes_fp64_v2<DV, DX, HESS>(v, x, t0, h, s_mid, mb, me, s, own_n);
  else
#endif
    nodes_fp64<DV, DX, HESS, CLAMP>(v, x, t0, h, s_mid, mb, me, s);
  // node n: t_n = t1 lies outside the eps-support (d(t1) < 0, FindZero
  // returns the outer end, R1), so its term is < 2^-52 of the peak term.
  // (Leaving node n out altogether from 64 bins, as the FP32 loop does,
  // measured 0.4% slower here: profiles/r02v_skipn.log.)
  if (own_n && !n_done) {
    if (n >= kEndF32MinBins) end_half_f32<DV, DX, HESS>(v, x, s_mid, fma((double)n, h, t0), s);
    else end_half_f64<DV, DX, HESS>(v, x, s_mid, fma((double)n, h, t0), s);
  }
  return s;
}

// ---------------------------------------------------------------- FP32 path
// FP32 entry point sums, returned in FP64: S2 (and S1) can exceed FLT_MAX
// where their ratio to S0, the output, does not.
struct Sums32 {
  double S0, S1, S2;
};

// FP32 entry point quadrature.  The weight exponent g(t) - s is a difference
// of terms as large as v t and x cosh t (~1e2 in config 4) whose FP32
// rounding (~1e-5 absolute) would reach the 1e-5 tolerance on log K near
// |log K| ~ 1 (measured by emulation: 9e-6 with FP32 recurrences for
// cosh t).  So the node position, cosh t and the exponent are formed in FP64
// (6 FP64 instructions per node) and rounded once to FP32, where MUFU.EX2
// takes the exponential; the weights, q, p and the three sums are FP32, the
// sums blocked every 16 nodes into FP64 (error ~1e-7 ~ eps32).
// double -> float by truncation with three integer ops (IADD, SHF.L.U64,
// LOP3) instead of F2F.F32.F64, which runs on the XU pipe next to MUFU and
// made the FP32 kernel XU-bound.  Valid for |d| in [2^-100, 2^127]; smaller
// magnitudes give 0 (a weight exponent of 0 +- 2^-100 is 1 to FP32 anyway).
__device__ __forceinline__ float d2f_trunc(double d) {
  const int hi = __double2hiint(d), lo = __double2loint(d);
  const int b = hi - 0x38000000;                        // rebias exponent 1023 -> 127
  int f;
  asm("shf.l.clamp.b32 %0, %1, %2, 3;" : "=r"(f) : "r"(lo), "r"(b));   // (b << 3) | (lo >> 29)
  f = (f & 0x7fffffff) | (hi & 0x80000000);
  return (hi & 0x7ff00000) < 0x39b00000 ? 0.0f : __int_as_float(f);
}

template <bool DV, bool DX>
__device__ __forceinline__ Sums32 quad_f32(float vf, float xf, float t0f, float hf, float shift,
                                           int n, int mb, int me) {
  const double kLog2e = 1.4426950408889634;
  const double v = vf, x = xf, t0 = t0f, h = hf;
  // exponent in log2 units: a2 = (v t - x cosh t - s - log 2) log2(e)
  const double v2 = v * kLog2e, nx2 = -x * kLog2e;
  const double ns2 = -((double)shift + kLn2) * kLog2e;
  const double eh = exp(h), ehi = rcp64(eh);
  const int sig = max(0, (int)ceil(fma((double)n, h, t0) * kLog2e) - 64);
  const double sc_sig = ldexp(1.0, sig), sc_inv = ldexp(1.0, -sig);
  const float ehf = float(eh), ehif = float(ehi);
  const float m2vl = float(-2.0 * v2);
  const float eqf = ex2_approx(m2vl * hf);
  const float a1 = -expm1f(-2.0f * vf * hf);
  double S0 = 0.0, S1 = 0.0, S2 = 0.0;
  static_assert(kAnchor % 4 == 0, "anchor interval must hold whole groups");
#pragma unroll 1
  for (int c0 = mb; c0 < me; c0 += kAnchor) {
    const int c1 = min(c0 + kAnchor, me);
    double tc = fma((double)c0, h, t0);
    double et = 0.5 * exp(tc), eti = 0.25 * rcp64(et);
    const float tcf = float(tc);
    // FP32 copies of t and e^{+-t}/2 for the products (weights only)
    float etf = float(et * sc_inv), etif = float(eti * sc_inv);   // 2^-sig scaled (see v2)
    float q = ex2_approx(m2vl * tcf);                      // q, p re-anchored per chunk
    float p = -expm1f(-2.0f * vf * tcf);
    float B0 = 0.0f, B1 = 0.0f, B2 = 0.0f;                 // per-chunk FP32 partial sums
    int m = c0;
    float jf = 0.0f;
#pragma unroll 1
    for (; m + 4 <= c1; m += 4) {
      double ch[4], tt[4];
      float E[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        tt[j] = j == 0 ? tc : fma(double(j), h, tc);
        ch[j] = et + eti;
        et *= eh;
        eti *= ehi;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) E[j] = ex2_approx(d2f_trunc(fma(nx2, ch[j], fma(v2, tt[j], ns2))));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float chf = etf + etif;
        const float tf = fmaf(jf + float(j), hf, tcf);
        const float w = fmaf(E[j], q, E[j]);               // E (1 + q)
        B0 += w;
        if (DX) B2 = fmaf(w, chf, B2);
        if (DV) {
          B1 = fmaf(E[j] * tf, p, B1);
          p = fmaf(q, a1, p);
        }
        q *= eqf;
        etf *= ehf;
        etif *= ehif;
      }
      jf += 4.0f;
      tc = fma((double)(m + 4), h, t0);
    }
#pragma unroll 1
    for (; m < c1; ++m) {
      const double t = fma((double)m, h, t0);
      const double ch = et + eti;
      et *= eh;
      eti *= ehi;
      const float E = ex2_approx(d2f_trunc(fma(nx2, ch, fma(v2, t, ns2))));
      const float w = fmaf(E, q, E);
      B0 += w;
      if (DX) B2 = fmaf(w, etf + etif, B2);
      if (DV) {
        B1 = fmaf(E * float(t), p, B1);
        p = fmaf(q, a1, p);
      }
      q *= eqf;
      etf *= ehf;
      etif *= ehif;
    }
    S0 += B0; S1 += B1; S2 += double(B2) * sc_sig;
  }
  // half weights of nodes 0 and n, evaluated directly
  auto half_node = [&](int mm) {
    const double t = fma((double)mm, h, t0);
    const double et = 0.5 * exp(t);
    const double ch = et + 0.25 * rcp64(et);
    const float E = 0.5f * ex2_approx(float(fma(nx2, ch, fma(v2, t, ns2))));
    const float tf = float(t);
    const float q1 = ex2_approx(m2vl * tf);
    const float w = fmaf(E, q1, E);
    S0 -= w;
    if (DX) S2 -= double(w) * ch;
    if (DV) S1 -= double(E * tf) * (-expm1f(-2.0f * vf * tf));
  };
  if (mb == 0) half_node(0);
  if (mb < me && me == n + 1) half_node(n);
  return Sums32{S0, S1, S2};
}

// FP32 entry point, fixed-point exponent.  The weight exponent in log2 units,
// a2 = (v t - x cosh t - s - log 2) log2(e), is formed in FP64 as
// A = a2 + 126 + M with M = 1.5 * 2^29 (ulp 2^-23), so the low word of A is
// ((n + 126) << 23) | f for a2 = n + f/2^23 (n = floor(a2), two's complement).
// Then 2^(a2) = 2^n * 2^(f/2^23) costs one LOP3 (the float 1.f), one MUFU.EX2
// (2^(1.f) = 2 * 2^(f/2^23)) and one IADD3 on its bits: ex2 + lo - bits(1.f)
// = bits(2^(f/2^23)) + (n << 23) -- no FP64->FP32 conversion, no shift.
// Needs a2 in [-126, 128): the caller takes this path only when the range's
// end points sit less than 60 (natural log) below the peak.  Quantisation of
// a2 to 2^-23 (plus two FP64 roundings at that scale) is <= 1.2e-7 relative
// in a weight, below FP32 rounding.
__device__ __forceinline__ float exp2_fixed(double A) {
  const int lo = __double2loint(A);
  int fb;   // (lo & 0x007fffff) | 0x3f800000 as one LOP3 (lut 0xEA = (a & b) | c)
  asm("lop3.b32 %0, %1, 0x007fffff, %2, 0xEA;" : "=r"(fb) : "r"(lo), "r"(0x3f800000));
  const float e = ex2_approx(__int_as_float(fb));
  return __int_as_float(__float_as_int(e) + lo - fb);
}


// FP32 entry point, group-base form (v3).  The FP64 fixed-point exponent
// (exp2_fixed above; round 1 formed it at every node) is formed once per group
// of 4 nodes, at the group's first node
// c: A_c = v2 t_c - X_c + cst (X = x cosh t log2(e) = Xp + Xm, Xp/m =
// (x log2(e)/2) e^{+-t}; 7 FP64 operations), E_c = 2^{a2_c} by exp2_fixed.
// The other nodes j = 1..3 of the group differ from it by an exponent that
// is small in magnitude and is formed in FP32 from FP32 copies of Xp_c, Xm_c:
//   a2_{c+j} - a2_c = j v2 h - dX_j,  dX_j = Xp_c (e^{jh} - 1) + Xm_c (e^{-jh} - 1),
// E_{c+j} = E_c 2^{j v2 h - dX_j} (MUFU.EX2 and one FMUL).  Its FP32 rounding
// is ~1e-7 (x cosh t) 3h in log2 units: < 3e-7 on config 4, < 3e-6 in the
// cancellation band x ~ 0.66 v ~ 1e4 (test_wide_domain_fuzz_f32*).  cosh t
// at every node is X_c + dX_j (S2 is sum w X, scaled by 1/(x log2(e)) once),
// so the e^{+-t} FP32 recurrences of v2 go away.  Xp_c, Xm_c step per group
// as X + X u (u = e^{+-4h} - 1, one FFMA2) and, with q, p and t, are
// re-anchored from FP64 every kBlk3 nodes, where the FP32 partial sums are
// also added into FP64 (every 128 nodes: FP32 recurrence drift over 32 group
// steps is a few ulp, the partial sums' rounding ~1e-7 relative).  ~44
// instructions per 4 nodes against 60 for v2.
// e^x for the FP32 entry point's FP64 recurrence states (x in [-700, 700]):
// 2^(x log2 e) with n = rint by the 1.5 2^52 magic add, e^(f ln 2), |f| <= 1/2,
// by its Taylor series to degree 11 (truncation < 3e-15 relative; the
// reduction's rounding ~1e-16 |x|): ~16 FP64 operations against ~35
// instructions and a slow-path branch for libdevice exp.  The recurrences it
// seeds need ~1e-11 (the FP32 weights resolve ~1e-7 of an exponent <= 10^3).
__device__ __forceinline__ double exp_seed64(double x) {
  const double y = x * 1.4426950408889634;
  const double M = 6755399441055744.0;
  const double t = y + M;
  const double f = (y - (t - M)) * 0.6931471805599453;
  double p = fma(f, 1.0 / 39916800.0, 1.0 / 3628800.0);
  p = fma(p, f, 1.0 / 362880.0);
  p = fma(p, f, 1.0 / 40320.0);
  p = fma(p, f, 1.0 / 5040.0);
  p = fma(p, f, 1.0 / 720.0);
  p = fma(p, f, 1.0 / 120.0);
  p = fma(p, f, 1.0 / 24.0);
  p = fma(p, f, 1.0 / 6.0);
  p = fma(p, f, 0.5);
  p = fma(p, f, 1.0);
  p = fma(p, f, 1.0);
  return __hiloint2double(__double2hiint(p) + (__double2loint(t) << 20), __double2loint(p));
}

#ifndef BLK_F32_BLK3
#define BLK_F32_BLK3 128
#endif
template <bool DV, bool DX>
__device__ __forceinline__ Sums32 quad_f32_v3(float vf, float xf, float t0f, float hf, float shift,
                                              int n, int mb, int me) {
  constexpr int G = 4, CH = BLK_F32_BLK3;
  static_assert(CH % G == 0, "blocks hold whole groups");
  const double kLog2e = 1.4426950408889634;
  const double v = vf, x = xf, t0 = t0f, h = hf;
  const double v2 = v * kLog2e;
  const double hx2 = 0.5 * x * kLog2e;
  const double cst = (805306368.0 + 126.0) - ((double)shift + kLn2) * kLog2e;
  const double e1 = exp_seed64(h), e1i = rcp64(e1), e2 = e1 * e1, eG = e2 * e2, eGi = rcp64(eG);
  const double e2i = e1i * e1i;
  // per-lane FP32 constants of the group offsets
  const float U1 = float(e1 - 1.0), U2 = float(e2 - 1.0), U3 = float(e2 * e1 - 1.0);
  const float V1 = float(e1i - 1.0), V2 = float(e2i - 1.0), V3 = float(e2i * e1i - 1.0);
  const float uG = float(eG - 1.0), uGi = float(eGi - 1.0);
  const double v2h = v2 * h;
  const float J1 = float(v2h), J2 = float(2.0 * v2h), J3 = float(3.0 * v2h);
  const float m2vl = float(-2.0 * v2);
  const float eq1 = ex2_approx(m2vl * hf), eq2 = eq1 * eq1, eq3 = eq2 * eq1, eq4 = eq2 * eq2;
  // 1 - q^j from a1 = 1 - q by exact identities (no cancellation for small
  // v h, R21): 1 - q^2 = a1 (2 - a1), 1 - q^3 = a1 + q (1 - q^2), 1 - q^4 = a2 (2 - a2)
  const float a1 = -expm1f(-2.0f * vf * hf), a2 = a1 * (2.0f - a1);
  const float a3 = fmaf(1.0f - a1, a2, a1), a4 = a2 * (2.0f - a2);
  const float h4 = 4.0f * hf;
  const double tb = fma((double)mb, h, t0);
  const double ebx = exp_seed64(tb);
  double XpG = hx2 * ebx, XmG = hx2 * rcp64(ebx);
  const double XpB = XpG, XmB = XmG;          // node mb (for node 0's half weight)
  double S0 = 0.0, S1 = 0.0, S2 = 0.0;
  float qn0 = 0.0f, pn0 = 0.0f;
  bool n_done = false;
  // node n lies outside the eps = 2^-23 support (R1): from 64 bins its half
  // weight (< 2^-24 of the peak term) is below the FP32 resolution of S0 and
  // it is not evaluated (c4 +2.9%, profiles/r02v_skipn.log)
  const bool skip_n = n >= kEndF32MinBins && me == n + 1;
  const int mend = skip_n ? n : me;
  double md = (double)mb;
  int m = mb;
#pragma unroll 1
  while (m < mend) {
    const int c1 = min(m + CH, mend);
    const double tcd = fma(md, h, t0);
    const float tcf = float(tcd);
    // FP32 state re-anchored per block: Xp, Xm, q = e^{-2vt}, p = 1 - q, t
    float2 X2 = f2(float(XpG), float(XmG));
    const float q0 = ex2_approx(m2vl * tcf);
    const float p0 = -expm1f(-2.0f * vf * tcf);
    if (m == 0) { qn0 = q0; pn0 = p0; }        // node 0's q, p for its half weight
    float2 qA = f2(q0, q0 * eq1), qB = f2(q0 * eq2, q0 * eq3);
    float2 pA = f2(p0, fmaf(q0, a1, p0)), pB = f2(fmaf(q0, a2, p0), fmaf(q0, a3, p0));
    float2 tA = f2(tcf, tcf + hf), tB = f2(fmaf(2.0f, hf, tcf), fmaf(3.0f, hf, tcf));
    float2 C0 = f2s(0.0f), C1 = f2s(0.0f), C2 = f2s(0.0f);
#pragma unroll 1
    for (; m + G <= c1; m += G) {
      const double tc = fma(md, h, t0);
      md += (double)G;
      const float Ec = exp2_fixed(fma(v2, tc, cst) - (XpG + XmG));
      XpG *= eG; XmG *= eGi;
      // exponent offsets of nodes 1..3 from the group's first node
      const float Xp = X2.x, Xm = X2.y;
      const float dX1 = fmaf(Xp, U1, Xm * V1);
      const float2 dX23 = fma2(f2s(Xp), f2(U2, U3), mul2(f2s(Xm), f2(V2, V3)));
      const float E1 = Ec * ex2_approx(J1 - dX1);
      const float2 E23 = mul2(f2s(Ec), ex2_2(add2(f2(J2, J3), mul2(dX23, f2s(-1.0f)))));
      const float Xc = Xp + Xm;
      const float2 XA = f2(Xc, Xc + dX1), XB = add2(f2s(Xc), dX23);
      X2 = fma2(X2, f2(uG, uGi), X2);
      const float2 EA = f2(Ec, E1);
      const float2 wA = fma2(EA, qA, EA), wB = fma2(E23, qB, E23);   // E (1 + q)
      C0 = add2(C0, add2(wA, wB));
      if (DX) C2 = fma2(wB, XB, fma2(wA, XA, C2));
      if (DV) {
        C1 = fma2(mul2(EA, pA), tA, C1);
        C1 = fma2(mul2(E23, pB), tB, C1);
        pA = fma2(qA, f2s(a4), pA);
        pB = fma2(qB, f2s(a4), pB);
      }
      qA = mul2(qA, f2s(eq4));
      qB = mul2(qB, f2s(eq4));
      tA = add2(tA, f2s(h4));
      tB = add2(tB, f2s(h4));
    }
    float B0 = C0.x + C0.y, B1 = C1.x + C1.y, B2 = C2.x + C2.y;
    float q = qA.x, p = pA.x, tf = tA.x;
#pragma unroll 1
    for (; m < c1; ++m) {                                // remainder, one node at a time
      const double t = fma(md, h, t0);
      md += 1.0;
      const double X = XpG + XmG;
      // node n carries weight 1/2, applied here
      n_done = (m == n);
      const float E = exp2_fixed(fma(v2, t, cst) - X) * (n_done ? 0.5f : 1.0f);
      XpG *= e1; XmG *= e1i;
      const float w = fmaf(E, q, E);
      B0 += w;
      if (DX) B2 = fmaf(w, float(X), B2);
      if (DV) B1 = fmaf(E * tf, p, B1);
      if (DV) p = fmaf(q, a1, p);
      q *= eq1;
      tf += hf;
    }
    S0 += B0; S1 += B1; S2 += B2;
  }
  // half weights of nodes 0 and n.  Node 0's is taken back here
  // from the exact start state and the first block's q, p (its t is t0f);
  // node n's was applied in the remainder loop when it ended there (always
  // for one lane and n + 1 not a multiple of 4, e.g. n = 128), else it is
  // taken back here, X one step back from the final recurrence state.
  if (mb == 0) {
    const double X = XpB + XmB;
    const float E = 0.5f * exp2_fixed(fma(v2, t0, cst) - X);
    const float w = fmaf(E, qn0, E);
    S0 -= w;
    if (DX) S2 -= double(w) * X;
    if (DV) S1 -= double(E * t0f) * pn0;
  }
  if (mb < me && me == n + 1 && !n_done && !skip_n) {
    const double X = fma(XpG, e1i, XmG * e1);
    const double t = fma((double)n, h, t0);
    const float E = 0.5f * exp2_fixed(fma(v2, t, cst) - X);
    const float tf1 = float(t);
    const float q1 = ex2_approx(m2vl * tf1);
    const float w = fmaf(E, q1, E);
    S0 -= w;
    if (DX) S2 -= double(w) * X;
    if (DV) S1 -= double(E * tf1) * (-expm1f(-2.0f * vf * tf1));
  }
  return Sums32{S0, S1, S2 * (1.0 / (2.0 * hx2))};
}

}  // namespace blk
