// logk_quad.cuh -- fixed-bin trapezoid quadrature in log-sum-exp form
// (PAPER.md Eq. (int)) with the derivative integrands of Sec. 4.1
// accumulated in the same pass over f's nodes (R14).
//
// With shift s ~ g(t_p) and q = e^{-2vt}:
//   exp(g(t) - s)                 = E (1 + q),   E = exp(vt - x cosh t - s - log 2)
//   t tanh(vt) exp(g(t) - s)      = E t (1 - q)
//   cosh t exp(g(t) - s)          = E (1 + q) cosh t
// so one exponential per node carries all three sums.  e^{+-t} and q advance
// by geometric recurrences (re-anchored every kAnchor nodes for e^{+-t});
// p = 1 - q advances additively, p' = p + q (1 - e^{-2vh}), which has no
// cancellation for small vt (R21).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "logk_range.cuh"

namespace blk {

constexpr int kExpTab = 256;      // 2^(j/256), j = 0..255, in shared memory
constexpr int kAnchor = 32;       // FP64 re-anchoring interval for e^{+-t}

// exp(a) for a in [-707, 709] by Tang's table method: a = (k/256) ln2 + r,
// |r| <= ln2/512, exp(a) = 2^(k>>8) * T[k&255] * (1 + r + r^2/2 + r^3/6 + r^4/24).
// Inputs below -707 are clamped (the weight is < 1e-307 of the peak there).
// ~10 FP64-pipe instructions + 1 LDS.64 + 3 integer ops.
__device__ __forceinline__ double exp_tab(double a, const double *__restrict__ tab) {
  const double kInvL = 369.3299304675746;             // 256 / ln 2
  const double kMagic = 6755399441055744.0;            // 1.5 * 2^52: round-to-int trick
  const double kC1 = 0.00270760617331689;              // ln2/256 to 32 bits: k*kC1 exact
  const double kC2 = 7.453964567463233e-13;            // ln2/256 - kC1
  a = fmax(a, -707.0);
  double kd = fma(a, kInvL, kMagic);
  const int k = __double2loint(kd);
  kd -= kMagic;
  double r = fma(kd, -kC1, a);                         // Cody-Waite reduction
  r = fma(kd, -kC2, r);
  double p = fma(r, 4.1666666666666666e-02, 1.6666666666666666e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r * r, r);
  double tj = tab[k & (kExpTab - 1)];
  double res = fma(tj, p, tj);
  int hi = __double2hiint(res) + ((k >> 8) << 20);
  return __hiloint2double(hi, __double2loint(res));
}

// Same as exp_tab but safe for any finite a (anchors: t itself may be large).
__device__ __forceinline__ double exp_anchor(double a, const double *__restrict__ tab) {
  return a > 709.0 ? (double)INFINITY : exp_tab(a, tab);
}

// Fill the 2^(j/256) table (block-cooperative; caller syncs).
__device__ __forceinline__ void fill_exp_table(double *tab) {
  for (int j = threadIdx.x; j < kExpTab; j += blockDim.x) tab[j] = exp2((double)j / kExpTab);
}

struct Sums64 {
  double S0, S1, S2;
};

// Nodes m in [mb, me) of the n-interval trapezoid on [t0, t0 + n h]; node 0
// and node n carry weight 1/2 via a log-2 larger shift.
template <bool DV, bool DX>
__device__ __forceinline__ Sums64 quad_f64(double v, double x, double t0, double h,
                                           double shift, int n, int mb, int me,
                                           const double *__restrict__ tab) {
  Sums64 s{0.0, 0.0, 0.0};
  const double s_mid = shift + kLn2;          // E = exp(vt - x cosh t - s_mid)
  const double s_end = s_mid + kLn2;          // half weight
  const double eh = exp(h), ehi = exp(-h);
  const double m2v = -2.0 * v;
  double tb = fma((double)mb, h, t0);
  double q = exp(m2v * tb);                   // q_m = e^{-2 v t_m}
  const double eq = exp(m2v * h);
  double p = -expm1(m2v * tb);                // p_m = 1 - q_m without cancellation
  const double a1 = -expm1(m2v * h);
  const int cnt = me - mb;
  if (cnt <= 0) return s;
  const int nch = (cnt + kAnchor - 1) / kAnchor;
  const int csz = (cnt + nch - 1) / nch;
#pragma unroll 1
  for (int c0 = mb; c0 < me; c0 += csz) {
    const int c1 = min(c0 + csz, me);
    double t = fma((double)c0, h, t0);
    double et = 0.5 * exp_anchor(t, tab);     // e^t / 2
    double eti = 0.5 * exp_tab(-t, tab);      // e^-t / 2
#pragma unroll 4
    for (int m = c0; m < c1; ++m) {
      const double ch = et + eti;             // cosh t
      const double sm = (m == 0 || m == n) ? s_end : s_mid;
      const double arg = fma(-x, ch, fma(v, t, -sm));
      const double E = exp_tab(arg, tab);
      const double w = fma(E, q, E);          // E (1 + q)
      s.S0 += w;
      if (DX) s.S2 = fma(w, ch, s.S2);
      if (DV) s.S1 = fma(E * t, p, s.S1);
      if (DV) p = fma(q, a1, p);
      q *= eq;
      t += h;
      et *= eh;
      eti *= ehi;
    }
  }
  return s;
}

// ---------------------------------------------------------------- FP32 path
struct Sums32 {
  float S0, S1, S2;
};

// exp(a) with the argument split so that ex2.approx sees an exactly
// representable a*log2(e) (hi) and the rounding residue (lo) is applied to
// first order: relative error ~2 ulp instead of |a| ulp.
__device__ __forceinline__ float exp_split_f32(float a) {
  const float kL2e = 1.4426950408889634f;
  const float kL2eLo = 1.9259629911266175e-08f;       // log2(e) - kL2e
  float y = a * kL2e;
  float yl = fmaf(a, kL2e, -y);
  yl = fmaf(a, kL2eLo, yl);
  float e = ex2_approx(y);
  return fmaf(e, yl * 0.6931471805599453f, e);
}

template <bool DV, bool DX>
__device__ __forceinline__ Sums32 quad_f32(float v, float x, float t0, float h, float shift,
                                           int n, int mb, int me) {
  Sums32 s{0.0f, 0.0f, 0.0f};
  const float kL2e = 1.4426950408889634f;
  const float s_mid = shift + 0.6931471805599453f;
  const float s_end = s_mid + 0.6931471805599453f;
  const float m2v = -2.0f * v;
  const float a1 = -expm1f(m2v * h);
  float p = -expm1f(m2v * fmaf((float)mb, h, t0));
  float mf = (float)mb;
  // partial sums per block of 16 nodes keep FP32 accumulation error small
  Sums32 blk{0.0f, 0.0f, 0.0f};
  int inblk = 0;
#pragma unroll 2
  for (int m = mb; m < me; ++m) {
    const float t = fmaf(mf, h, t0);
    const float e = exp_split_f32(t);
    const float ch = 0.5f * (e + rcp_approx(e));
    const float q = ex2_approx(m2v * kL2e * t);
    const float sm = (m == 0 || m == n) ? s_end : s_mid;
    const float arg = fmaf(-x, ch, fmaf(v, t, -sm));
    const float E = ex2_approx(arg * kL2e);
    const float w = fmaf(E, q, E);
    blk.S0 += w;
    if (DX) blk.S2 = fmaf(w, ch, blk.S2);
    if (DV) blk.S1 = fmaf(E * t, p, blk.S1);
    if (DV) p = fmaf(q, a1, p);
    mf += 1.0f;
    if (++inblk == 16) {
      s.S0 += blk.S0; s.S1 += blk.S1; s.S2 += blk.S2;
      blk = Sums32{0.0f, 0.0f, 0.0f};
      inblk = 0;
    }
  }
  s.S0 += blk.S0; s.S1 += blk.S1; s.S2 += blk.S2;
  return s;
}

}  // namespace blk
