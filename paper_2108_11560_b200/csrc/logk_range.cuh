// logk_range.cuh -- per-element integration plan (range finding) on sm_100a.
//
// Alg. 1 FindRange, Alg. 2 FindZero and lines 2-9 of Alg. 3 (PAPER.md
// P:144-218), with the readings recorded in DESIGN.md §3
// (R1 orientation F(a) < 0 <= F(b), return a; R3 clip to [a, mid];
// R4 at most 10 iterations, the "until" clause on working tolerances;
// R5 lo = t_s when m = 0; R5b brackets from the shape of g in the FP32
// finder; R18 Newton with F'(a)=0 -> bisection point).  Independent of
// oracle/ (no shared code).
//
// Two implementations:
//   * PlanF32: FP32 FMA pipe + MUFU (ex2/lg2/rcp.approx).  The two point
//     evaluations of one FindZero iteration (at the bisection point and at the
//     Newton point) are independent, so they run as packed f32x2 operations
//     (FFMA2/FADD2/FMUL2, sm_100) -- half the issue slots.  The plan only has
//     to be conservative at the log-eps level (R20), so finding it
//     in FP32 leaves the FP64 pipe to the quadrature.  Used from 48 bins (the
//     FP32 entry point: from 16) inside its safe domain.
//   * PlanF64 / PlanF64Tab: double -- the paper's working-precision variant
//     with Alg. 1 as printed, stopping only once converged (the oracle's
//     ranges); used for coarse grids, outside the FP32-safe domain and on
//     request (BLK_RANGE_F64).
// Every point evaluation returns F and F' jointly (they share e^t, e^-t and
// q = e^{-2vt}).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace blk {

constexpr int kMaxIter = 10;     // Alg. 2
constexpr int kRangeCap = 11;    // FindRange doubling cap: t <= t_s + 2^12
constexpr double kLn2 = 0.69314718055994530942;
constexpr double kLogEpsF64 = -36.043653389117154;   // log 2^-52 (R9)
constexpr double kLogEpsF32 = -15.942385152878742;   // log 2^-23 (R9)

__device__ __forceinline__ float ex2_approx(float a) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}
__device__ __forceinline__ float lg2_approx(float a) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}
__device__ __forceinline__ float rcp_approx(float a) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float a) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}
#ifndef BLK_SMART_FAST
#define BLK_SMART_FAST 1
#endif
// Quotients and square roots of the R5b bracket guesses: every guess is
// checked by evaluating F there, so MUFU approximations (2 instructions)
// serve instead of IEEE division / sqrt (~10 with the FCHK slow-path branch).
__device__ __forceinline__ float guess_div(float a, float b) {
  return BLK_SMART_FAST ? a * rcp_approx(b) : a / b;
}
__device__ __forceinline__ float guess_sqrt(float a) {
  return BLK_SMART_FAST ? sqrt_approx(a) : sqrtf(a);
}

// ------------------------------------------------------------ packed helpers
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2s(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 ex2_2(float2 a) { return f2(ex2_approx(a.x), ex2_approx(a.y)); }
__device__ __forceinline__ float2 lg2_2(float2 a) { return f2(lg2_approx(a.x), lg2_approx(a.y)); }
__device__ __forceinline__ float2 rcp_2(float2 a) { return f2(rcp_approx(a.x), rcp_approx(a.y)); }

// Result of the range finding for one element.
template <class T>
struct Plan {
  T tp, gp, t0, t1;
  T dmin;     // min of d = g - g(t_p) - log eps at t0 and t1 (for the exp-clamp decision)
  bool ok;
};

// ============================================================== FP32 (packed)
struct PlanF32 {
  static constexpr float kL2e = 1.4426950408889634f;
  static constexpr float kLn2f = 0.6931471805599453f;
  float v, x, hx, v2, m2vs, L;

  // F = g'(t) = v tanh(vt) - x sinh t,  F' = g''(t) = v^2 sech^2(vt) - x cosh t
  // (Eq. 4-5);  tanh = (1-q)/(1+q), sech^2 = 4q/(1+q)^2, q = e^{-2vt}.
  __device__ __forceinline__ void peak1(float t, float &F, float &dF) const {
    float e = ex2_approx(t * kL2e), ei = rcp_approx(e);
    float q = ex2_approx(m2vs * t), r = rcp_approx(1.0f + q);
    F = v * ((1.0f - q) * r) - hx * (e - ei);
    dF = v2 * (4.0f * q * r * r) - hx * (e + ei);
  }
  __device__ __forceinline__ void peak2(float2 t, float2 &F, float2 &dF) const {
    float2 e = ex2_2(mul2(t, f2s(kL2e)));
    float2 ei = rcp_2(e);
    float2 q = ex2_2(mul2(t, f2s(m2vs)));
    float2 r = rcp_2(add2(q, f2s(1.0f)));
    float2 th = mul2(add2(f2s(1.0f), mul2(q, f2s(-1.0f))), r);
    float2 s2 = mul2(mul2(q, f2s(4.0f)), mul2(r, r));
    F = fma2(f2s(v), th, mul2(f2s(-hx), add2(e, mul2(ei, f2s(-1.0f)))));
    dF = fma2(f2s(v2), s2, mul2(f2s(-hx), add2(e, ei)));
  }
  // F = d(t) = g(t) - g(t_p) - log eps, F' = g'(t);
  // g(t) = vt + log(1+q) - log 2 - x cosh t, c = g(t_p) + log eps + log 2.
  __device__ __forceinline__ void thr1(float c, float t, float &F, float &dF) const {
    float e = ex2_approx(t * kL2e), ei = rcp_approx(e);
    float q = ex2_approx(m2vs * t), r = rcp_approx(1.0f + q);
    F = v * t + lg2_approx(1.0f + q) * kLn2f - hx * (e + ei) - c;
    dF = v * ((1.0f - q) * r) - hx * (e - ei);
  }
  __device__ __forceinline__ void thr2(float c, float2 t, float2 &F, float2 &dF) const {
    float2 e = ex2_2(mul2(t, f2s(kL2e)));
    float2 ei = rcp_2(e);
    float2 q = ex2_2(mul2(t, f2s(m2vs)));
    float2 opq = add2(q, f2s(1.0f));
    float2 r = rcp_2(opq);
    float2 lq = lg2_2(opq);
    float2 base = fma2(lq, f2s(kLn2f), f2s(-c));
    base = fma2(f2s(v), t, base);
    F = fma2(f2s(-hx), add2(e, ei), base);
    float2 omq = add2(f2s(1.0f), mul2(q, f2s(-1.0f)));
    dF = fma2(mul2(f2s(v), omq), r, mul2(f2s(-hx), add2(e, mul2(ei, f2s(-1.0f)))));
  }
  __device__ __forceinline__ float gval(float t) const {
    float e = ex2_approx(t * kL2e), ei = rcp_approx(e);
    float q = ex2_approx(m2vs * t);
    return v * t + lg2_approx(1.0f + q) * kLn2f - float(kLn2) - hx * (e + ei);
  }
};

// One FindZero iteration, shared by both precisions: bisection
// point mid, clipped Newton point tn (R2, R3, R18) ...
template <class T>
__device__ __forceinline__ void fz_points(T a, T Fa, T dFa, T b, T &mid, T &tn) {
  mid = a + (b - a) * T(0.5);                    // t_shrink
  T t = a - Fa / dFa;                            // t_newton from the current a (R2)
  t = isfinite(t) ? t : mid;                     // F'(a) = 0 or overflow (R18)
  T lo = fmin(a, mid), hi = fmax(a, mid);        // Clip to [a, mid] (R3)
  tn = fmin(fmax(t, lo), hi);
}
// FP32 variant with the search direction known at compile time: ASC (t0
// search, a = 0 < b = t_p) or descending (peak and t1 searches, a > b).  The
// clip to [a, mid] then needs two min/max, and a non-finite Newton point
// lands on mid through the NaN rules of fminf/fmaxf: NaN -> mid; +inf (only
// from F'(a) = +0, i.e. the first t0 step, R18) -> mid in the ascending
// search; -inf (F'(a) = -0) -> mid in the descending ones.  The remaining
// infinities (-inf ascending, +inf descending) need F(a)/F'(a) of the
// wrong sign, which the bracket invariants exclude.
template <bool ASC>
__device__ __forceinline__ void fz_points_f32(float a, float Fa, float dFa, float b, float &mid,
                                              float &tn) {
  mid = fmaf(b - a, 0.5f, a);
  const float t = fmaf(-Fa, rcp_approx(dFa), a);
  tn = ASC ? fmaxf(fminf(t, mid), a) : fminf(fmaxf(t, mid), a);
}

// ... then the three-way bracket update, branch-free.
template <class T>
__device__ __forceinline__ void fz_update(T mid, T tn, T Fm, T dFm, T Ft, T dFt, T &a, T &Fa,
                                          T &dFa, T &b) {
  const bool c1 = Fm < T(0);                     // zero in (mid, b)
  const bool c2 = Ft < T(0);                     // zero in (tn, mid)
  //                                                else zero in (a, tn)
  const T na = c1 ? mid : (c2 ? tn : a);
  const T nFa = c1 ? Fm : (c2 ? Ft : Fa);
  const T ndFa = c1 ? dFm : (c2 ? dFt : dFa);
  b = c1 ? b : (c2 ? mid : tn);
  a = na; Fa = nFa; dFa = ndFa;
}

// Alg. 2 with the two evaluations packed into f32x2 operations.  The loop
// ends after max_iter = 10 iterations or earlier, per the paper's
// "until" clause, on a working tolerance in log units (R4; the
// literal tol = 1 on |a_i - a_{i-1}| stops on the first iteration that keeps
// a and breaks config 3):
//   * range ends (F = d = g - g_p - log eps): once the kept end a -- still on
//     the outer side, F(a) < 0 is invariant -- has F(a) >= -end_nats, i.e.
//     the integrand there is at least e^-end_nats of the eps level.  The
//     range is then conservative and wider than the exact one by end_nats /
//     |g'| at each end (~end_nats/36 of the half-width for a quadratic peak).
//     (A test on the Newton correction relative to |a - t_p| instead would
//     stop AT FindRange's end where d grows like x cosh t: there F/F' ~ 1 is
//     small against the probe distance, leaving ranges many times too wide.)
//   * the peak (F = g', F' = g''): what matters is not where t_p is but how
//     far g(a) lies below the maximum, because g(t_p) becomes the log-sum-exp
//     shift and the base of the eps threshold: Newton's estimate of that gap
//     is F(a)^2 / (2 |F'(a)|), and the search stops once it is below
//     peak_gap.  (A relative criterion on t_p would leave gaps of
//     |g''| (tol t_p)^2 / 2 -- over 100 for x ~ 1e-30 and v ~ 1e4.)
// The tolerances follow the grid (the FP32 finder only runs from 48 bins,
// kF32PlanMinBins).  From 128 bins the FP64 trapezoid is insensitive to the
// range -- widening the ends by 50% changes no output beyond 7e-14 (SURVEY
// A.4) -- so end_nats = 8, peak_gap = 4 (the ends then lie at most ~12 nats
// beyond the eps level, ~1/3 of the half-width): c3 +4.6%, c2 +3.9%, c5 +2.8%
// against the relative 2^-8 rule, outputs unchanged to rounding
// (profiles/r02g_endnats.log, profiles/r02t_e8.log); 48-127 bins can still
// carry a discretisation error on extreme inputs that a wider range shifts,
// so 0.1 and 1/64.  The FP32 entry point's threshold is eps = 2^-23 (R9), an
// eps-support about half as wide, over which 64 nodes leave the trapezoid far
// below FP32 rounding (converged from 16 nodes): 8 and 4 from 64
// bins (c4 +13%), the 0.1 / 1/64 tier at 16-63.
struct FzTol {
  float end_nats;   // range ends: stop once F(a) >= -end_nats
  float peak_gap;   // peak: stop once F^2 / (2|F'|) <= peak_gap
};
#ifndef BLK_END_NATS_128
#define BLK_END_NATS_128 8.0f
#endif
#ifndef BLK_PEAK_GAP_128
#define BLK_PEAK_GAP_128 4.0f
#endif
__host__ __device__ __forceinline__ FzTol fz_tol_for(int nbins) {
  return nbins >= 128 ? FzTol{BLK_END_NATS_128, BLK_PEAK_GAP_128} : FzTol{0.1f, 0.015625f};
}
__host__ __device__ __forceinline__ FzTol fz_tol_f32_entry(int nbins) {
  return nbins >= 64 ? FzTol{BLK_END_NATS_128, BLK_PEAK_GAP_128} : FzTol{0.1f, 0.015625f};
}
template <bool PEAK, bool ASC, class PF>
__device__ __forceinline__ float find_zero_f32(const PF &P, float c, float a, float &Fa,
                                               float &dFa, float b, FzTol tol) {
#pragma unroll 2
  for (int i = 0; i < kMaxIter; ++i) {
    if (PEAK) {
      // (an overflowed F'(a) -- far FindRange probes at x cosh t > FP32_MAX --
      // carries no information and must not end the search)
      if (Fa * Fa <= (2.0f * tol.peak_gap) * fabsf(dFa) && fabsf(dFa) <= 3.0e38f) break;
    } else {
      if (Fa >= -tol.end_nats) break;
    }
    float mid, tn;
    fz_points_f32<ASC>(a, Fa, dFa, b, mid, tn);
    float2 F, dF;
    if (PEAK) P.peak2(f2(mid, tn), F, dF);
    else P.thr2(c, f2(mid, tn), F, dF);
    fz_update<float>(mid, tn, F.x, dF.x, F.y, dF.y, a, Fa, dFa, b);
  }
  return a;
}

// Alg. 1 FindRange from t_s with F(t_s) >= 0.  Returns false when
// the doubling cap is exceeded.  (lo, hi) bracket the zero with F(hi) < 0;
// F(hi), F'(hi) are returned for the first Newton step of FindZero.
template <class Fn, class T>
__device__ __forceinline__ bool find_range(const Fn &f, T ts, T &lo, T &hi, T &Fhi, T &dFhi) {
  int m = 0;
  T step = T(2);
  f(ts + step, Fhi, dFhi);
#pragma unroll 1
  while (Fhi >= T(0)) {
    if (++m > kRangeCap) return false;
    step = step * T(2);
    f(ts + step, Fhi, dFhi);
  }
  lo = (m == 0) ? ts : ts + step * T(0.5);
  hi = ts + step;
  return true;
}

// Alg. 3 lines 2-9 in FP32.  The regime test g''(0) = v^2 - x > 0
// is taken in double on the caller's inputs.  SMART (every kernel's
// FP32 range finder): the brackets Alg. 2 starts from come from the shape of
// g instead of Alg. 1's
// doubling from t_s (R5b) -- every bracket end is checked by
// evaluating F, and Alg. 1 runs whenever a check fails, so the results are
// ranges Alg. 2 could have returned from Alg. 1's brackets:
//   peak: [0, t*], t* = asinh(v/x): g'(0) = 0 and g'(t*) = v (tanh(v t*) - 1) <= 0;
//   t0:   a Newton step of d from t_p - dq (normally inside: the left flank is
//         flatter than the quadratic model) lands outside next to the root
//         (d is concave there), dq = sqrt(2 |log eps| / |g''(t_p)|);
//   t1:   likewise from t_p + 0.7 dq (the right flank falls faster than the
//         model), or t_p + 0.7 dq itself when it is already outside.
// c3 +9.9%, c2 +5.6%, c4 (FP32 entry point) +14% (profiles/r02y_smart*.log,
// profiles/r02zb_peak.log).
#ifndef BLK_T1_FRAC
#define BLK_T1_FRAC 0.7f
#endif
#ifndef BLK_T0_FRAC
#define BLK_T0_FRAC 1.0f
#endif
// R5b bracket helpers (see above).  Each returns whether its bracket was
// established; the caller falls back to Alg. 1 otherwise.
template <class PFN>
__device__ __forceinline__ bool smart_peak_bracket(const PlanF32 &P, const PFN &pf, float &lo,
                                                   float &hi, float &Fh, float &dFh) {
  // t* = asinh(v/x) is always on the outer side of the peak:
  // g'(t*) = v (tanh(v t*) - 1) <= 0, and for v t* >> 1 it is the peak to
  // FP32 resolution.  [0, t*] brackets it (g'(0) = 0).  (t* is moved out by
  // 2^-10 relative + 1e-4: where v t* >> 1, g'(t*) is below the FP32
  // rounding of its two ~v-sized terms and could test >= 0.)
  const float z = guess_div(P.v, P.x);
  const float ta = z > 1e4f ? lg2_approx(2.0f * z) * PlanF32::kLn2f
                            : lg2_approx(z + guess_sqrt(fmaf(z, z, 1.0f))) * PlanF32::kLn2f;
  const float ts = fmaf(ta, 1.0009765625f, 1e-4f);
  pf(ts, Fh, dFh);
  if (!(Fh < 0.0f && isfinite(dFh))) return false;
  hi = ts; lo = 0.0f;
  return true;
}
// t0: the left flank is flatter than the quadratic model (g'' -> v^2 sech^2 -
// x cosh t rises towards 0), so t_p - dq is normally inside: one Newton step
// from it lands outside (d is concave, its tangent lies above it) next to the
// root, and [tz, t_p - dq] brackets the root for Alg. 2.
template <class DFN>
__device__ __forceinline__ void smart_t0_bracket(const DFN &df, float tp, float dq, float &a,
                                                 float &Fa, float &dFa, float &b) {
  const float tq = tp - BLK_T0_FRAC * dq;
  if (!(tq > 0.0f)) return;
  float Fq, dFq;
  df(tq, Fq, dFq);
  if (Fq < 0.0f) { a = tq; Fa = Fq; dFa = dFq; }
  else if (dFq > 0.0f) {
    const float tz = fmaxf(tq - guess_div(Fq, dFq), 0.0f);
    float Fz, dFz;
    df(tz, Fz, dFz);
    if (Fz < 0.0f) { a = tz; Fa = Fz; dFa = dFz; b = tq; }
  }
}
// t1: the right flank falls faster than the model (x cosh t), so t_p + 0.7 dq
// is outside or a Newton step from it (inside) lands outside.
template <class DFN>
__device__ __forceinline__ bool smart_t1_bracket(const DFN &df, float tp, float dq, float &lo,
                                                 float &hi, float &Fh, float &dFh) {
  const float tq = tp + BLK_T1_FRAC * dq;
  df(tq, Fh, dFh);
  if (Fh < 0.0f) { hi = tq; lo = tp; return true; }
  if (dFh < 0.0f) {
    const float tz = tq - guess_div(Fh, dFh);
    float Fz, dFz;
    df(tz, Fz, dFz);
    if (Fz < 0.0f && isfinite(dFz)) { hi = tz; lo = tq; Fh = Fz; dFh = dFz; return true; }
  }
  return false;
}
// half-width of the quadratic model g ~ g_p - K (t - t_p)^2 / 2 at the eps
// level, when usable for the brackets (< 32 keeps every probe in FP32 range)
__device__ __forceinline__ float model_halfwidth(float L, float K) {
  const float dq = guess_sqrt(guess_div(-2.0f * L, K));
  return (isfinite(dq) && dq > 0.0f && dq < 32.0f) ? dq : 0.0f;
}

template <bool SMART = false>
__device__ __forceinline__ Plan<float> make_plan_f32(double vd, double xd, double log_eps,
                                                    FzTol tol) {
  Plan<float> p;
  PlanF32 P;
  P.v = float(vd); P.x = float(xd); P.hx = 0.5f * P.x; P.v2 = P.v * P.v;
  P.m2vs = -2.0f * P.v * PlanF32::kL2e; P.L = float(log_eps);
  float lo, hi, Fh, dFh;
  p.ok = false;
  p.tp = 0.0f;
  float K;                         // |g''| at the peak (curvature for the range brackets)
  auto pf = [&](float t, float &F, float &dF) { P.peak1(t, F, dF); };
  if (vd * vd - xd > 0.0) {
    const bool br = SMART && smart_peak_bracket(P, pf, lo, hi, Fh, dFh);
    if (!br && !find_range(pf, 0.0f, lo, hi, Fh, dFh)) return p;
    p.tp = find_zero_f32<true, false>(P, 0.0f, hi, Fh, dFh, lo, tol);  // (t_e, t_s)
    K = fabsf(dFh);
  } else {
    K = P.x - P.v2;                // -g''(0) in the monotone regime
  }
  p.gp = P.gval(p.tp);
  const float c = p.gp + P.L + float(kLn2);
  auto df = [&](float t, float &F, float &dF) { P.thr1(c, t, F, dF); };
  const float dq = SMART ? model_halfwidth(P.L, K) : 0.0f;
  p.t0 = 0.0f;
  float d0 = -P.x - p.gp - P.L;                                    // d(0)
  if (d0 <= 0.0f) {
    float a = 0.0f, Fa = d0, dFa = 0.0f, b = p.tp;
    if (dq > 0.0f) smart_t0_bracket(df, p.tp, dq, a, Fa, dFa, b);
    p.t0 = find_zero_f32<false, true>(P, c, a, Fa, dFa, b, tol);
    d0 = Fa;
  }
  const bool br = dq > 0.0f && smart_t1_bracket(df, p.tp, dq, lo, hi, Fh, dFh);
  if (!br && !find_range(df, p.tp, lo, hi, Fh, dFh)) return p;
  p.t1 = find_zero_f32<false, false>(P, c, hi, Fh, dFh, lo, tol);
  p.dmin = fminf(d0, Fh);
  p.ok = true;
  return p;
}

// Alg. 2 for the range ends with the search direction a runtime flag (ASC:
// the t0 search from a = 0 up to t_p; otherwise the t1 search down from the
// FindRange end), so that two lanes can run the t0 and the t1 search of the
// same element in one loop (make_plan_f32_pair).  Same updates and stopping
// rule as find_zero_f32<false, ASC>.
template <class PF>
__device__ __forceinline__ float find_zero_f32_rt(const PF &P, float c, float a, float &Fa,
                                                  float dFa, float b, FzTol tol,
                                                  bool asc, bool active) {
#pragma unroll 1
  for (int i = 0; active && i < kMaxIter; ++i) {
    if (Fa >= -tol.end_nats) break;
    const float mid = fmaf(b - a, 0.5f, a);
    const float t = fmaf(-Fa, rcp_approx(dFa), a);
    const float tn = asc ? fmaxf(fminf(t, mid), a) : fminf(fmaxf(t, mid), a);
    float2 F, dF;
    P.thr2(c, f2(mid, tn), F, dF);
    fz_update<float>(mid, tn, F.x, dF.x, F.y, dF.y, a, Fa, dFa, b);
  }
  return a;
}

// make_plan_f32 for a PAIR of lanes working on the same element (lanes per
// element >= 2): both find t_p and g(t_p); then the even lane runs the t0
// search while the odd lane runs FindRange + the t1 search
// in the same loop, and the two exchange their ends with a
// shuffle.  Same ranges as make_plan_f32 (the same arithmetic per search);
// the latency of one of the two searches is saved, which is what bounds
// small batches.  All lanes of the pair must be active.
template <bool SMART = false>
__device__ __forceinline__ Plan<float> make_plan_f32_pair(double vd, double xd, double log_eps,
                                                         FzTol tol, bool odd) {
  Plan<float> p;
  PlanF32 P;
  P.v = float(vd); P.x = float(xd); P.hx = 0.5f * P.x; P.v2 = P.v * P.v;
  P.m2vs = -2.0f * P.v * PlanF32::kL2e; P.L = float(log_eps);
  float lo, hi, Fh, dFh;
  p.ok = false;
  p.tp = 0.0f;
  float K;
  bool peak_ok = true;
  if (vd * vd - xd > 0.0) {
    auto pf = [&](float t, float &F, float &dF) { P.peak1(t, F, dF); };
    const bool br = SMART && smart_peak_bracket(P, pf, lo, hi, Fh, dFh);
    peak_ok = br || find_range(pf, 0.0f, lo, hi, Fh, dFh);
    if (peak_ok) p.tp = find_zero_f32<true, false>(P, 0.0f, hi, Fh, dFh, lo, tol);
    K = fabsf(dFh);
  } else {
    K = P.x - P.v2;
  }
  // (both lanes of the pair reach the shuffles below, also on failure)
  p.gp = P.gval(p.tp);
  const float c = p.gp + P.L + float(kLn2);
  const float d0 = -P.x - p.gp - P.L;                             // d(0)
  const float dq = SMART ? model_halfwidth(P.L, K) : 0.0f;
  auto df = [&](float t, float &F, float &dF) { P.thr1(c, t, F, dF); };
  bool range_ok = peak_ok;
  float a, Fa, dFa, b;
  bool active;
  if (odd) {                                                      // t1: FindRange first
    if (range_ok) {
      const bool br = dq > 0.0f && smart_t1_bracket(df, p.tp, dq, lo, hi, Fh, dFh);
      range_ok = br || find_range(df, p.tp, lo, hi, Fh, dFh);
    }
    a = hi; Fa = Fh; dFa = dFh; b = lo; active = range_ok;
  } else {                                                        // t0 from 0 (if needed)
    a = 0.0f; Fa = d0; dFa = 0.0f; b = p.tp; active = range_ok && d0 <= 0.0f;
    if (active && dq > 0.0f) smart_t0_bracket(df, p.tp, dq, a, Fa, dFa, b);
  }
  a = find_zero_f32_rt(P, c, a, Fa, dFa, b, tol, !odd, active);
  // the two lanes of the pair, named explicitly: they may leave the search
  // loop at different iterations, and __shfl_xor_sync with this mask waits
  // for both (an __activemask() taken here could miss the partner)
  const unsigned mask = 3u << ((threadIdx.x & 31u) & ~1u);
  const float a_o = __shfl_xor_sync(mask, a, 1);
  const float Fa_o = __shfl_xor_sync(mask, Fa, 1);
  const bool ok_o = __shfl_xor_sync(mask, (int)range_ok, 1) != 0;
  const float t0 = odd ? a_o : a, t1 = odd ? a : a_o;
  const float F0 = odd ? Fa_o : Fa, F1 = odd ? Fa : Fa_o;
  if (!peak_ok || !(odd ? range_ok : ok_o)) return p;
  p.t0 = (d0 <= 0.0f) ? t0 : 0.0f;
  p.t1 = t1;
  p.dmin = fminf(d0 <= 0.0f ? F0 : d0, F1);
  p.ok = true;
  return p;
}

// ==================================================================== FP64
struct PlanF64 {
  double v, x, hx, v2, m2v;
  __device__ __forceinline__ void peak(double t, double &F, double &dF) const {
    double e = exp(t), ei = 1.0 / e;
    double q = exp(m2v * t), r = 1.0 / (1.0 + q);
    F = v * ((1.0 - q) * r) - hx * (e - ei);
    dF = v2 * (4.0 * q * r * r) - hx * (e + ei);
  }
  __device__ __forceinline__ void thr(double c, double t, double &F, double &dF) const {
    double e = exp(t), ei = 1.0 / e;
    double q = exp(m2v * t), r = 1.0 / (1.0 + q);
    F = v * t + log1p(q) - hx * (e + ei) - c;
    dF = v * ((1.0 - q) * r) - hx * (e - ei);
  }
  __device__ __forceinline__ double gval(double t) const {
    double e = exp(t), ei = 1.0 / e;
    return v * t + log1p(exp(m2v * t)) - kLn2 - hx * (e + ei);
  }
};

// Alg. 2 in double.  The paper's working-precision variant: it stops only
// once a has converged (Newton correction below 2^-45 of the scale: |a| for
// the peak, |a - t_p| for the range ends), where further iterations leave a
// unchanged to the last bits -- so the ranges are those of the oracle's fixed
// 10 iterations (BLK_RANGE_F64 reproduces the oracle at coarse grids, R20).
template <class Fn>
__device__ __forceinline__ double find_zero_f64(const Fn &f, double a, double &Fa, double dFa,
                                                double b, double ref) {
#pragma unroll 1
  for (int i = 0; i < kMaxIter; ++i) {
    const double rhs = 2.842170943040401e-14 * fabs((a - ref) * dFa);   // 2^-45
    if (fabs(Fa) <= rhs && rhs <= 1e300) break;
    double mid, tn;
    fz_points<double>(a, Fa, dFa, b, mid, tn);
    double Fm, dFm, Ft, dFt;
    f(mid, Fm, dFm);
    f(tn, Ft, dFt);
    fz_update<double>(mid, tn, Fm, dFm, Ft, dFt, a, Fa, dFa, b);
  }
  return a;
}

// Alg. 3 lines 2-9 in double for a point-evaluation type PF (peak, thr, gval).
template <class PF>
__device__ __forceinline__ Plan<double> make_plan_f64_with(const PF &P, double v, double x,
                                                         double log_eps) {
  Plan<double> p;
  double lo, hi, Fh, dFh;
  p.ok = false;
  p.tp = 0.0;
  auto pf = [&](double t, double &F, double &dF) { P.peak(t, F, dF); };
  if (v * v - x > 0.0) {
    if (!find_range(pf, 0.0, lo, hi, Fh, dFh)) return p;
    p.tp = find_zero_f64(pf, hi, Fh, dFh, lo, 0.0);
  }
  p.gp = P.gval(p.tp);
  const double c = p.gp + log_eps + kLn2;
  auto df = [&](double t, double &F, double &dF) { P.thr(c, t, F, dF); };
  p.t0 = 0.0;
  double d0 = -x - p.gp - log_eps;
  if (d0 <= 0.0) p.t0 = find_zero_f64(df, 0.0, d0, 0.0, p.tp, p.tp);
  if (!find_range(df, p.tp, lo, hi, Fh, dFh)) return p;
  p.t1 = find_zero_f64(df, hi, Fh, dFh, lo, p.tp);
  p.dmin = fmin(d0, Fh);
  p.ok = true;
  return p;
}

// libdevice point evaluations (kernels without the shared exp table)
__device__ __forceinline__ Plan<double> make_plan_f64(double v, double x, double log_eps) {
  return make_plan_f64_with(PlanF64{v, x, 0.5 * x, v * v, -2.0 * v}, v, x, log_eps);
}

// Inputs for which the FP32 range finder is used under BLK_RANGE_AUTO:
// e^t, x cosh t and g stay far inside FP32 range and the d(t) cancellation
// error stays below ~0.1 in log units.
// (for v, x >= 0 the IEEE bit patterns order like the values: compared as
// 64-bit integers on the ALU, not as doubles on the FP64 pipe, which the other
// warps' node loops keep busy -- a DSETP there waits for it)
__device__ __forceinline__ bool f32_plan_domain(double v, double x) {
  const long long xb = __double_as_longlong(x), vb = __double_as_longlong(v);
  return xb >= 0x39B4484BFEEBC2A0LL /* 1e-30 */ && xb <= 0x40C3880000000000LL /* 1e4 */ &&
         vb <= 0x40C3880000000000LL;
}
// Input test of every kernel (R16): x > 0 finite and v finite, by integer
// tests on the bit patterns (same reason as above).
__device__ __forceinline__ bool valid_input(double v, double x) {
  const long long xb = __double_as_longlong(x), vb = __double_as_longlong(v);
  return xb > 0 && xb < 0x7FF0000000000000LL && (vb & 0x7FFFFFFFFFFFFFFFLL) < 0x7FF0000000000000LL;
}

// DESIGN.md R23: ranges must end below t = 709 (e^t overflows double at
// 709.78, cosh t at 710.48); beyond, the element has no result (NaN), in the
// oracle as in the kernels.
constexpr double kTMax = 709.0;

// Below this many bins BLK_RANGE_AUTO also takes the FP64 range finder: a
// coarse grid's discretisation error depends on where the nodes fall, so
// only the paper's working-precision ranges reproduce the oracle there
// (R20); from it on the grid has converged (n = 48
// within 2.4e-15 / 2.1e-14 of mpmath on every config) and the result is
// insensitive to the range: with the FP32 finder at 48-63 bins every config
// stays within 0.05 of the north_star tolerance of the oracle element by
// element, as the FP64 finder does, and runs 6x faster (48 bins: 1.16e10
// against 1.85e9 evals/s on c3; at 32 bins c1 and c4 would not converge --
// profiles/r02zt_coarse_auto.log).
#ifndef BLK_F32_PLAN_MIN_BINS
#define BLK_F32_PLAN_MIN_BINS 48
#endif
constexpr int kF32PlanMinBins = BLK_F32_PLAN_MIN_BINS;

// The range finder BLK_RANGE_AUTO picks for one element.
__device__ __forceinline__ bool use_f32_plan(int range_mode, int nbins, double v, double x) {
  return range_mode == 0 && nbins >= kF32PlanMinBins && f32_plan_domain(v, x);
}
// The FP32 entry point (eps = 2^-23, R9) resolves only FP32: from 16 nodes over
// its eps-support the trapezoid error is below FP32 rounding for any
// conservative range (<= 1.3e-6 from n = 16), so its FP32 range
// finder serves from 16 bins (the 0.1-nat tier below 64), the FP64 one below.
constexpr int kF32EntryPlanMinBins = 16;
__device__ __forceinline__ bool use_f32_plan_f32_entry(int range_mode, int nbins, double v,
                                                       double x) {
  return range_mode == 0 && nbins >= kF32EntryPlanMinBins && f32_plan_domain(v, x);
}

}  // namespace blk
