// logk_range.cuh -- per-element integration plan (range finding) on sm_100a.
//
// Alg. 1 FindRange, Alg. 2 FindZero and lines 2-9 of Alg. 3 (PAPER.md
// P:144-218), with the readings recorded in DESIGN.md §3
// (R1 orientation F(a) < 0 <= F(b), return a; R3 clip to [a, mid];
// R4 fixed 10 iterations; R5 lo = t_s when m = 0; R18 Newton with F'(a)=0
// -> bisection point).  Independent of oracle/ (no shared code).
//
// Templated on the working type T and a math policy:
//   MathF32: FP32 FMA pipe + MUFU (ex2/lg2/rcp.approx).  The plan only needs
//            to be conservative at the log-eps level (R20), so the
//            range is found here and the quadrature (FP64 pipe) consumes it.
//   MathF64: libdevice double functions -- the paper's working-precision
//            variant, used outside the FP32-safe domain and on request.
// Every point evaluation returns F and F' jointly (they share e^t, e^-t and
// q = e^{-2vt}), so one FindZero iteration costs two joint evaluations.
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

struct MathF32 {
  using T = float;
  static constexpr float kLog2e = 1.4426950408889634f;
  static constexpr float kLn2f = 0.6931471805599453f;
  // exp(a) for an argument pre-multiplied by log2(e)
  __device__ __forceinline__ static float exp2s(float a2) { return ex2_approx(a2); }
  __device__ __forceinline__ static float scale(float a) { return a * kLog2e; }
  // log(1 + q), q in [0, 1]
  __device__ __forceinline__ static float log1p01(float q) { return lg2_approx(1.0f + q) * kLn2f; }
  __device__ __forceinline__ static float rcp(float a) { return rcp_approx(a); }
  __device__ __forceinline__ static float div(float a, float b) { return __fdividef(a, b); }
};

struct MathF64 {
  using T = double;
  __device__ __forceinline__ static double exp2s(double a) { return exp(a); }
  __device__ __forceinline__ static double scale(double a) { return a; }
  __device__ __forceinline__ static double log1p01(double q) { return log1p(q); }
  __device__ __forceinline__ static double rcp(double a) { return 1.0 / a; }
  __device__ __forceinline__ static double div(double a, double b) { return a / b; }
};

// F = g'(t) = v tanh(vt) - x sinh t,  F' = g''(t) = v^2 sech^2(vt) - x cosh t
// (Eq. 4-5).  tanh = (1-q)/(1+q), sech^2 = 4q/(1+q)^2, q = e^{-2vt}.
template <class M>
struct PeakFn {
  using T = typename M::T;
  T v, hx, v2, m2vs, ones;  // hx = x/2, v2 = v^2, m2vs = scale(-2v), ones = scale(1)
  __device__ __forceinline__ void operator()(T t, T &F, T &dF) const {
    T e = M::exp2s(ones * t);
    T ei = M::rcp(e);
    T q = M::exp2s(m2vs * t);
    T r = M::rcp(T(1) + q);
    T th = (T(1) - q) * r;
    T s2 = T(4) * q * r * r;
    F = v * th - hx * (e - ei);
    dF = v2 * s2 - hx * (e + ei);
  }
};

// F = d(t) = g(t) - g(t_p) - log eps,  F' = g'(t)
// g(t) = vt + log(1+q) - log 2 - x cosh t;  c = g(t_p) + log eps + log 2.
template <class M>
struct ThreshFn {
  using T = typename M::T;
  T v, hx, m2vs, ones, c;
  __device__ __forceinline__ void operator()(T t, T &F, T &dF) const {
    T e = M::exp2s(ones * t);
    T ei = M::rcp(e);
    T q = M::exp2s(m2vs * t);
    T r = M::rcp(T(1) + q);
    F = v * t + M::log1p01(q) - hx * (e + ei) - c;
    dF = v * (T(1) - q) * r - hx * (e - ei);
  }
};

// g(t) itself (Eq. 3), for g(t_p).
template <class M>
__device__ __forceinline__ typename M::T g_value(typename M::T v, typename M::T hx,
                                                 typename M::T m2vs, typename M::T ones,
                                                 typename M::T t) {
  using T = typename M::T;
  T e = M::exp2s(ones * t);
  T ei = M::rcp(e);
  T q = M::exp2s(m2vs * t);
  return v * t + M::log1p01(q) - T(kLn2) - hx * (e + ei);
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

// Alg. 2 FindZero, fixed kMaxIter iterations, F(a) < 0 <= F(b).
template <class M, class Fn, class T>
__device__ __forceinline__ T find_zero(const Fn &f, T a, T Fa, T dFa, T b) {
#pragma unroll 1
  for (int i = 0; i < kMaxIter; ++i) {
    T mid = a + (b - a) * T(0.5);                 // t_shrink
    T tn = a - M::div(Fa, dFa);                   // t_newton from the current a (R2)
    if (!isfinite(tn)) tn = mid;                  // F'(a) = 0 (R18)
    T lo = fmin(a, mid), hi = fmax(a, mid);       // Clip to [a, mid] (R3)
    tn = fmin(fmax(tn, lo), hi);
    T Fm, dFm, Ft, dFt;
    f(mid, Fm, dFm);
    f(tn, Ft, dFt);
    if (Fm < T(0)) {
      a = mid; Fa = Fm; dFa = dFm;
    } else if (Ft < T(0)) {
      b = mid; a = tn; Fa = Ft; dFa = dFt;
    } else {
      b = tn;
    }
  }
  return a;
}

// Alg. 3 lines 2-9: t_p, g(t_p), t0, t1 in type M::T.
// The regime test g''(0) = v^2 - x > 0 is taken in double on the
// caller's inputs.  Returns false when FindRange hits its cap.
template <class M>
__device__ __forceinline__ bool make_plan(double vd, double xd, double log_eps,
                                          typename M::T &tp, typename M::T &gp,
                                          typename M::T &t0, typename M::T &t1) {
  using T = typename M::T;
  const T v = T(vd), x = T(xd);
  const T hx = T(0.5) * x;
  const T ones = M::scale(T(1));
  const T m2vs = M::scale(T(-2) * v);
  const T L = T(log_eps);
  T lo, hi, Fh, dFh;
  tp = T(0);
  if (vd * vd - xd > 0.0) {
    PeakFn<M> pf{v, hx, v * v, m2vs, ones};
    if (!find_range(pf, T(0), lo, hi, Fh, dFh)) return false;
    tp = find_zero<M>(pf, hi, Fh, dFh, lo);       // (t_e, t_s)
  }
  gp = g_value<M>(v, hx, m2vs, ones, tp);
  ThreshFn<M> df{v, hx, m2vs, ones, gp + L + T(kLn2)};
  t0 = T(0);
  const T d0 = -x - gp - L;                       // d(0) = g(0) - g(t_p) - log eps
  if (d0 <= T(0)) t0 = find_zero<M>(df, T(0), d0, T(0), tp);   // P:262-265, g'(0) = 0
  if (!find_range(df, tp, lo, hi, Fh, dFh)) return false;
  t1 = find_zero<M>(df, hi, Fh, dFh, lo);
  return true;
}

// Inputs for which the FP32 range finder is used under BLK_RANGE_AUTO:
// e^t, x cosh t and g stay far inside FP32 range and the d(t) cancellation
// error stays below ~0.1 in log units.
__device__ __forceinline__ bool f32_plan_domain(double v, double x) {
  return x >= 1e-30 && x <= 1e4 && v <= 1e4;
}

}  // namespace blk
