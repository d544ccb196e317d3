// logk_kernels.cu -- fused sm_100a kernels and the C ABI (include/bessel_logk.h).
//
// One kernel per precision does the whole hot path for its elements
// (SURVEY.md §8(a) a1-a7): load + canonicalise, regime test, peak, t0, t1
// (logk_range.cuh), fixed-bin quadrature with the three sums
// (logk_quad.cuh), epilogue log/divide, store.  No shared state besides the
// 16 KB exp table per block of the FP64 kernels; no atomics.  LPE (lanes per element) > 1 splits
// the n+1 nodes of one element across LPE adjacent lanes (every lane derives
// the identical plan) and combines the sums with warp shuffles.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "../../include/bessel_logk.h"
#include "logk_quad.cuh"
#include "logk_range.cuh"
#include "logk_nig.cuh"
#include "logk_io.cuh"
#ifdef BLK_DIAG
#include "logk_split.cuh"   // diagnostics build only (tools/): the two phases as two kernels
#endif

namespace blk {

constexpr int kDefaultThreads = 128;

#ifdef BLK_TIMELINE
// Diagnostic build only (tools/build_variants.py ...=BLK_TIMELINE): per-warp
// %globaltimer stamps (start, plan done, end) and SM id of the FP64 kernel.
constexpr int kTlMax = 1 << 16;
__device__ unsigned long long g_tl[kTlMax][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define BLK_TL(slot)                                                              \
  do {                                                                            \
    const unsigned w_ = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;             \
    if ((threadIdx.x & 31) == 0 && w_ < kTlMax) {                                 \
      g_tl[w_][slot] = gtimer();                                                  \
      if (slot == 0) g_tl[w_][3] = smid();                                        \
    }                                                                             \
  } while (0)
#else
#define BLK_TL(slot) do {} while (0)
#endif

template <int LPE, class T>
__device__ __forceinline__ T group_sum(T a) {
#pragma unroll
  for (int o = 1; o < LPE; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

// Bins [mb, me) handled by lane `sub` of LPE lanes for n+1 nodes.
template <int LPE>
__device__ __forceinline__ void lane_bins(int n, int sub, int &mb, int &me) {
  const int per = (n + 1 + LPE - 1) / LPE;
  mb = min(sub * per, n + 1);
  me = min(mb + per, n + 1);
}

#ifndef BLK_SMART_F64
#define BLK_SMART_F64 true
#endif
#ifndef BLK_SMART_F32
#define BLK_SMART_F32 true
#endif
// a2-a5 for one canonical element (v >= 0, x > 0 finite) of the FP64 entry
// point: the range finder BLK_RANGE_AUTO / BLK_RANGE_F64 selects (FP32 from
// 48 bins inside its domain, else FP64 with the table exp, which needs
// g_exp_tab loaded), t_p, g(t_p), [t0, t1] and dmin.  Returns whether the plan
// is usable.  Shared by the fused kernels and the plan export, so
// bessel_logk_plan_f64 reports exactly the plan the quadrature uses.
template <int LPE>
__device__ __forceinline__ bool element_plan_f64(double v, double x, int nbins, int range_mode,
                                                 int sub, double &tp, double &gp, double &t0,
                                                 double &t1, double &dmin) {
  bool ok;
  if (use_f32_plan(range_mode, nbins, v, x)) {
    const Plan<float> p = (LPE >= 2) ? make_plan_f32_pair<BLK_SMART_F64>(v, x, kLogEpsF64, fz_tol_for(nbins), sub & 1)
                                     : make_plan_f32<BLK_SMART_F64>(v, x, kLogEpsF64, fz_tol_for(nbins));
    ok = p.ok; tp = p.tp; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
  } else {
    const Plan<double> p = make_plan_f64_tab(v, x, kLogEpsF64);
    ok = p.ok; tp = p.tp; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
  }
  // R23: a range reaching t = kTMax (709; e^t overflows at 709.78) cannot be
  // integrated in double -- no result, as in the oracle (the FP32 finder's
  // domain, x >= 1e-30, keeps t1 far below it)
  return ok && isfinite(t1) && isfinite(gp) && t1 > t0 && t1 < kTMax;
}

// One element (or one lane of LPE) of the FP64 path after the exp table is
// in shared memory: a1-a7 for (vraw, x); the caller stores the outputs.
template <bool LOGK, bool DV, bool DX, int LPE>
__device__ __forceinline__ void f64_element(double vraw, double x, int sub, int nbins,
                                            int range_mode, double &o_logk, double &o_dv,
                                            double &o_dx) {
  const double *tab = g_exp_tab;
  const bool valid = valid_input(vraw, x);
  const double v = fabs(vraw);
  const long long vbits = __double_as_longlong(vraw);
  const double sgn = (vbits < 0 && vbits != (long long)0x8000000000000000ULL) ? -1.0 : 1.0;  // v < 0 (-0 -> +1)

  // a2-a5: integration plan (t_p, g(t_p), t0, t1)
  double t0 = 0.0, t1 = 0.0, gp = 0.0, dmin = 0.0, tp = 0.0;
  const bool ok = valid && element_plan_f64<LPE>(v, x, nbins, range_mode, sub, tp, gp, t0, t1, dmin);
  BLK_TL(1);
  // a6: fixed-bin quadrature, three sums in one pass
  Sums64 s{0.0, 0.0, 0.0};
  const double h = (t1 - t0) * rcp64((double)nbins);   // h = (t1 - t0)/n
  if (ok) {
    int mb, me;
    lane_bins<LPE>(nbins, sub, mb, me);
    // exponent arguments stay above -707 unless the range reaches far below
    // the eps level (never on valid ranges; kept exact for safety)
    if (dmin > -600.0) s = quad_f64<DV, DX, false>(v, x, t0, h, gp, nbins, mb, me, tab);
    else s = quad_f64<DV, DX, true>(v, x, t0, h, gp, nbins, mb, me, tab);
  }
  if (LPE > 1) {
    s.S0 = group_sum<LPE>(s.S0);
    if (DV) s.S1 = group_sum<LPE>(s.S1);
    if (DX) s.S2 = group_sum<LPE>(s.S2);
  }
  BLK_TL(2);
  // a7: epilogue
  const double nanv = __longlong_as_double(0x7ff8000000000000ULL);
  const double r = rcp64(s.S0);
  if (LOGK) o_logk = ok ? gp + log_sum(h * s.S0) : nanv;
  if (DV) o_dv = ok ? sgn * (s.S1 * r) : nanv;
  if (DX) o_dx = ok ? -(s.S2 * r) : nanv;
}

// The FP64 kernel: one element per lane (or LPE lanes per element).  (Two to
// eight elements per thread in sequence, amortising the table copy and the
// block launch, measured 2-6% slower on c2/c3/c5: the block-by-block launch
// staggers the XU-bound plan and the FP64-bound quadrature across warps,
// profiles/r02j_ept.log.)  VEC (one element per lane only; the host selects it
// for BLK_KERNEL_VEC128 when every stream is 16-B aligned): 128-bit
// warp-cooperative loads and stores (logk_io.cuh) for warps of 32 in-range
// elements, the scalar path for the ragged last warp.
template <bool LOGK, bool DV, bool DX, int LPE, bool VEC = false>
__global__ void __launch_bounds__(128, BLK_MINB)
logk_f64_kernel(const double *__restrict__ vin, const double *__restrict__ xin, size_t n_el,
                double *__restrict__ logk, double *__restrict__ dlogk_dv,
                double *__restrict__ dlogk_dx, int nbins, int range_mode) {
  static_assert(!VEC || LPE == 1, "128-bit I/O needs one element per lane");
  BLK_TL(0);
  const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t i = gtid / LPE;
  const int sub = (int)(gtid % LPE);
  const bool live = i < n_el;
  // Lanes past the end still take part in the shuffles (full-warp masks).
  // The input loads are issued before the table copy and its barrier, which
  // hide their latency (it stalled every warp at its first use of x).
  double vraw = 1.0, x = 1.0;
  if constexpr (VEC) {
    __shared__ __align__(16) double s_io[kIoWarps * kIoPerWarp];
    const bool full = (gtid | 31) < n_el;   // warp-uniform
    // transposed before the table barrier: finishing it after the barrier
    // perturbs ptxas's node-loop schedule (-3.6% on c3, profiles/r02io_vec128_ab.log)
    if (full) io_load_finish(s_io, io_load_issue(vin, xin, i), i, vraw, x);
    else if (live) { vraw = vin[i]; x = xin[i]; }
    load_exp_table_sync();
    double o0, o1, o2;
    f64_element<LOGK, DV, DX, 1>(vraw, x, 0, nbins, range_mode, o0, o1, o2);
    if (full) {
      // the barrier separates the input reads of s_io from these writes
      io_store<double, LOGK, DV, DX, false>(s_io, i, o0, o1, o2, logk, dlogk_dv, dlogk_dx);
    } else if (live) {
      if (LOGK) logk[i] = o0;
      if (DV) dlogk_dv[i] = o1;
      if (DX) dlogk_dx[i] = o2;
    }
  } else {
    if (live) { vraw = vin[i]; x = xin[i]; }
    load_exp_table_sync();
    double o0, o1, o2;
    f64_element<LOGK, DV, DX, LPE>(vraw, x, sub, nbins, range_mode, o0, o1, o2);
    if (live && sub == 0) {
      if (LOGK) logk[i] = o0;
      if (DV) dlogk_dv[i] = o1;
      if (DX) dlogk_dx[i] = o2;
    }
  }
}

// Second derivatives in the same pass: the three
// second-order sums of Sec. 4.1 over f's range and nodes.  Outputs may each
// be NULL; all six sums are always formed.
template <int LPE>
__global__ void __launch_bounds__(128, BLK_MINB)
logk_f64_hess_kernel(const double *__restrict__ vin, const double *__restrict__ xin, size_t n_el,
                     double *__restrict__ logk, double *__restrict__ dv_out,
                     double *__restrict__ dx_out, double *__restrict__ dvv_out,
                     double *__restrict__ dxx_out, double *__restrict__ dvx_out, int nbins,
                     int range_mode) {
  const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t i = gtid / LPE;
  const int sub = (int)(gtid % LPE);
  const bool live = i < n_el;
  const double vraw = live ? vin[i] : 1.0;   // loads issued ahead of the table copy
  const double x = live ? xin[i] : 1.0;
  load_exp_table_sync();
  const bool valid = valid_input(vraw, x);
  const double v = fabs(vraw);
  const long long vbits = __double_as_longlong(vraw);
  const double sgn = (vbits < 0 && vbits != (long long)0x8000000000000000ULL) ? -1.0 : 1.0;  // v < 0 (-0 -> +1)
  double t0 = 0.0, t1 = 0.0, gp = 0.0, dmin = 0.0, tp = 0.0;
  const bool ok = valid && element_plan_f64<LPE>(v, x, nbins, range_mode, sub, tp, gp, t0, t1, dmin);
  Sums64 s{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const double h = (t1 - t0) * rcp64((double)nbins);
  if (ok) {
    int mb, me;
    lane_bins<LPE>(nbins, sub, mb, me);
    if (dmin > -600.0) s = quad_f64<true, true, false, true>(v, x, t0, h, gp, nbins, mb, me, g_exp_tab);
    else s = quad_f64<true, true, true, true>(v, x, t0, h, gp, nbins, mb, me, g_exp_tab);
  }
  if (LPE > 1) {
    s.S0 = group_sum<LPE>(s.S0); s.S1 = group_sum<LPE>(s.S1); s.S2 = group_sum<LPE>(s.S2);
    s.S11 = group_sum<LPE>(s.S11); s.S22 = group_sum<LPE>(s.S22); s.S12 = group_sum<LPE>(s.S12);
  }
  if (!live || sub != 0) return;
  const double nanv = __longlong_as_double(0x7ff8000000000000ULL);
  const double r = rcp64(s.S0);
  const double m1 = s.S1 * r, m2 = s.S2 * r;
  if (logk) logk[i] = ok ? gp + log_sum(h * s.S0) : nanv;
  if (dv_out) dv_out[i] = ok ? sgn * m1 : nanv;
  if (dx_out) dx_out[i] = ok ? -m2 : nanv;
  if (dvv_out) dvv_out[i] = ok ? fma(-m1, m1, s.S11 * r) : nanv;
  if (dxx_out) dxx_out[i] = ok ? fma(-m2, m2, s.S22 * r) : nanv;
  if (dvx_out) dvx_out[i] = ok ? sgn * fma(m1, m2, -(s.S12 * r)) : nanv;
}

// The plan alone (bessel_logk_plan_f64): what the FP64 entry point integrates
// over for the same nbins and range_mode; NaN where it has no usable plan.
__global__ void __launch_bounds__(128)
logk_plan_f64_kernel(const double *__restrict__ vin, const double *__restrict__ xin, size_t n_el,
                     double *__restrict__ tp_out, double *__restrict__ gp_out,
                     double *__restrict__ t0_out, double *__restrict__ t1_out, int nbins,
                     int range_mode) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double vraw = i < n_el ? vin[i] : 1.0;
  const double x = i < n_el ? xin[i] : 1.0;
  load_exp_table_sync();
  if (i >= n_el) return;
  const bool valid = valid_input(vraw, x);
  double t0 = 0.0, t1 = 0.0, gp = 0.0, dmin = 0.0, tp = 0.0;
  const bool ok = valid && element_plan_f64<1>(fabs(vraw), x, nbins, range_mode, 0, tp, gp, t0, t1, dmin);
  const double nanv = __longlong_as_double(0x7ff8000000000000ULL);
  if (tp_out) tp_out[i] = ok ? tp : nanv;
  if (gp_out) gp_out[i] = ok ? gp : nanv;
  if (t0_out) t0_out[i] = ok ? t0 : nanv;
  if (t1_out) t1_out[i] = ok ? t1 : nanv;
}

#ifndef BLK_F32_EPT
#define BLK_F32_EPT 2   // FP32 kernel: elements per thread (2: +0.9% on c4, profiles/r02zv_f32_ept.log)
#endif
#ifndef BLK_F32_MINB
// FP32 entry point: 5 resident blocks per SM (96 registers; the v3 loop
// spills at 6 blocks / 80 registers: c4 -4%, profiles/r02e_f32v3.log)
#define BLK_F32_MINB 5
#endif
template <bool LOGK, bool DV, bool DX, int LPE>
__device__ __forceinline__ void f32_element(float vraw, float x, int sub, int nbins,
                                            int range_mode, float &o_logk, float &o_dv,
                                            float &o_dx) {
  const bool valid = (x > 0.0f) && isfinite(x) && isfinite(vraw);
  const float v = fabsf(vraw);
  const float sgn = (vraw < 0.0f) ? -1.0f : 1.0f;

  float t0 = 0.0f, t1 = 0.0f, gp = 0.0f, dmin = 0.0f;
  bool ok = false;
  if (valid) {
    if (use_f32_plan_f32_entry(range_mode, nbins, v, x)) {
      const Plan<float> p =
          (LPE >= 2) ? make_plan_f32_pair<BLK_SMART_F32>(v, x, kLogEpsF32, fz_tol_f32_entry(nbins), sub & 1)
                     : make_plan_f32<BLK_SMART_F32>(v, x, kLogEpsF32, fz_tol_f32_entry(nbins));
      ok = p.ok; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
    } else {
      const Plan<double> p = make_plan_f64(v, x, kLogEpsF32);
      ok = p.ok; t0 = (float)p.t0; t1 = (float)p.t1; gp = (float)p.gp; dmin = (float)p.dmin;
    }
    ok = ok && isfinite(t1) && isfinite(gp) && t1 > t0;
  }
  Sums32 s{0.0, 0.0, 0.0};
  const float h = (t1 - t0) * rcp_approx((float)nbins);   // the grid need not be IEEE-exact
  if (ok) {
    int mb, me;
    lane_bins<LPE>(nbins, sub, mb, me);
    // the fixed-point exponent needs every node within 2^-126 of the peak:
    // true when both range ends are < 60 below the log-eps level (always on
    // ranges found by Alg. 1-3; kept exact for safety)
    if (dmin > -60.0f) s = quad_f32_v3<DV, DX>(v, x, t0, h, gp, nbins, mb, me);
    else
      s = quad_f32<DV, DX>(v, x, t0, h, gp, nbins, mb, me);
  }
  if (LPE > 1) {
    s.S0 = group_sum<LPE>(s.S0);
    if (DV) s.S1 = group_sum<LPE>(s.S1);
    if (DX) s.S2 = group_sum<LPE>(s.S2);
  }
  const float nanv = __int_as_float(0x7fc00000);
  const double r0 = rcp64(s.S0);
  if (LOGK) o_logk = ok ? gp + logf(float(double(h) * s.S0)) : nanv;
  if (DV) o_dv = ok ? sgn * float(s.S1 * r0) : nanv;
  if (DX) o_dx = ok ? -float(s.S2 * r0) : nanv;
}

template <bool LOGK, bool DV, bool DX, int LPE, bool VEC = false>
__global__ void __launch_bounds__(128, BLK_F32_MINB)
logk_f32_kernel(const float *__restrict__ vin, const float *__restrict__ xin, size_t n_el,
                float *__restrict__ logk, float *__restrict__ dlogk_dv,
                float *__restrict__ dlogk_dx, int nbins, int range_mode) {
  static_assert(!VEC || LPE == 1, "128-bit I/O needs one element per lane");
  const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t i = gtid / LPE;
  const int sub = (int)(gtid % LPE);
  const bool live = i < n_el;
  float vraw = 1.0f, x = 1.0f;
  if constexpr (VEC) {
    __shared__ __align__(16) float s_io[kIoWarps * kIoPerWarp];
    const bool full = (gtid | 31) < n_el;   // warp-uniform
    if (full) io_load_finish(s_io, io_load_issue(vin, xin, i), i, vraw, x);
    else if (live) { vraw = vin[i]; x = xin[i]; }
    float o0, o1, o2;
    f32_element<LOGK, DV, DX, 1>(vraw, x, 0, nbins, range_mode, o0, o1, o2);
    if (full) {
      io_store<float, LOGK, DV, DX>(s_io, i, o0, o1, o2, logk, dlogk_dv, dlogk_dx);
    } else if (live) {
      if (LOGK) logk[i] = o0;
      if (DV) dlogk_dv[i] = o1;
      if (DX) dlogk_dx[i] = o2;
    }
  } else if (BLK_F32_EPT > 1 && LPE == 1) {
    // BLK_F32_EPT elements per thread, each next one's inputs loaded before the
    // current one is computed (their load latency hidden behind that work)
    size_t j = (size_t)blockIdx.x * blockDim.x * BLK_F32_EPT + threadIdx.x;
    float vn = 1.0f, xn = 1.0f;
    if (j < n_el) { vn = vin[j]; xn = xin[j]; }
#pragma unroll 1
    for (int e = 0; e < BLK_F32_EPT; ++e, j += blockDim.x) {
      const float vc = vn, xc = xn;
      if (e + 1 < BLK_F32_EPT && j + blockDim.x < n_el) { vn = vin[j + blockDim.x]; xn = xin[j + blockDim.x]; }
      float o0, o1, o2;
      f32_element<LOGK, DV, DX, 1>(vc, xc, 0, nbins, range_mode, o0, o1, o2);
      if (j < n_el) {
        if (LOGK) logk[j] = o0;
        if (DV) dlogk_dv[j] = o1;
        if (DX) dlogk_dx[j] = o2;
      }
    }
  } else {
    if (live) { vraw = vin[i]; x = xin[i]; }
    float o0, o1, o2;
    f32_element<LOGK, DV, DX, LPE>(vraw, x, sub, nbins, range_mode, o0, o1, o2);
    if (live && sub == 0) {
      if (LOGK) logk[i] = o0;
      if (DV) dlogk_dv[i] = o1;
      if (DX) dlogk_dx[i] = o2;
    }
  }
}

// ------------------------------------------------------------ microbenchmarks
constexpr int kMbChains = 8;

__global__ void mb_fp64_kernel(int iters, double *out) {
  double a[kMbChains];
  const double m = 1.0 + 1e-9 * threadIdx.x, c = 1e-12;
#pragma unroll
  for (int j = 0; j < kMbChains; ++j) a[j] = 1.0 + j * 1e-3 + blockIdx.x * 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < BLK_MB_UNROLL / kMbChains; ++u) {
#pragma unroll
      for (int j = 0; j < kMbChains; ++j) a[j] = fma(a[j], m, c);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < kMbChains; ++j) s += a[j];
  out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mb_fp32_kernel(int iters, float *out) {
  float a[kMbChains];
  const float m = 1.0f + 1e-7f * threadIdx.x, c = 1e-9f;
#pragma unroll
  for (int j = 0; j < kMbChains; ++j) a[j] = 1.0f + j * 1e-3f + blockIdx.x * 1e-6f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < BLK_MB_UNROLL / kMbChains; ++u) {
#pragma unroll
      for (int j = 0; j < kMbChains; ++j) a[j] = fmaf(a[j], m, c);
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < kMbChains; ++j) s += a[j];
  out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mb_mufu_kernel(int iters, float *out) {
  float a[kMbChains];
#pragma unroll
  for (int j = 0; j < kMbChains; ++j) a[j] = -1e-3f * (j + 1) - 1e-9f * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < BLK_MB_UNROLL / kMbChains; ++u) {
#pragma unroll
      for (int j = 0; j < kMbChains; ++j) a[j] = ex2_approx(a[j]) - 1.0f;
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < kMbChains; ++j) s += a[j];
  out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace blk

// ===================================================================== C ABI
namespace {

thread_local char g_err[256] = "";

blk_status fail(blk_status st, const char *msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return st;
}

blk_status cuda_fail(cudaError_t e, const char *where) {
  snprintf(g_err, sizeof g_err, "%s: %s", where, cudaGetErrorString(e));
  return BLK_ECUDA;
}

int auto_lanes(size_t n, int nbins) {
  // Small batches are latency-bound: splitting each element's nodes over a
  // few lanes shortens the quadrature (the range finding is repeated per
  // lane).  Measured on B200 (profiles/r01_lanes_small_batches.log, c2, 128
  // bins): it pays while n x lanes stays below ~40k threads, up to 8 lanes
  // (n = 1e3: 8 lanes 10 us vs 14; 1e4: 4 lanes; 2e4: 2; >= 3e4: 1).
  const size_t fill = 40000;
  int lanes = 1;
  while (lanes < 8 && n * lanes * 2 <= fill && (nbins + 1) / (lanes * 2) >= 8) lanes *= 2;
  return lanes;
}

template <class T>
blk_status validate(const T *v, const T *x, size_t n, const void *o1, const void *o2,
                    const void *o3, int nbins, const blk_options *opts, int &lanes,
                    int &mode, int &threads, int &kernel) {
  lanes = 0; mode = BLK_RANGE_AUTO; threads = blk::kDefaultThreads; kernel = BLK_KERNEL_AUTO;
  if (opts) {
    lanes = opts->lanes_per_element;
    mode = opts->range_mode;
    kernel = opts->kernel;
    if (opts->block_threads) threads = opts->block_threads;
  }
  if (kernel != BLK_KERNEL_AUTO && kernel != BLK_KERNEL_SIMPLE && kernel != BLK_KERNEL_VEC128)
    return fail(BLK_EINVAL, "bad kernel variant");
  if (kernel == BLK_KERNEL_VEC128 && lanes > 1)
    return fail(BLK_EINVAL, "BLK_KERNEL_VEC128 needs lanes_per_element 0 or 1");
  if (nbins < 2 || nbins > BLK_MAX_NBINS) return fail(BLK_EINVAL, "nbins out of range [2, 65536]");
  if (n > 0 && !o1 && !o2 && !o3) return fail(BLK_EINVAL, "all outputs are NULL");
  if (n > 0 && (!v || !x)) return fail(BLK_EINVAL, "v or x is NULL");
  if (mode != BLK_RANGE_AUTO && mode != BLK_RANGE_F64) return fail(BLK_EINVAL, "bad range_mode");
  if (lanes < 0 || lanes > 32 || (lanes & (lanes - 1))) return fail(BLK_EINVAL, "lanes_per_element must be 0 or a power of two <= 32");
  if (threads < 32 || threads > 128 || threads % 32) return fail(BLK_EINVAL, "block_threads must be a multiple of 32 in [32, 128]");
  if (n > ((size_t)1 << 40)) return fail(BLK_EINVAL, "n too large");
  if (kernel == BLK_KERNEL_VEC128) {
    lanes = 1;
    const uintptr_t m = (uintptr_t)v | (uintptr_t)x | (uintptr_t)o1 | (uintptr_t)o2 | (uintptr_t)o3;
    if (m & 15u) kernel = BLK_KERNEL_SIMPLE;   // scalar I/O, identical results
    return BLK_OK;
  }
  kernel = BLK_KERNEL_SIMPLE;
  if (lanes == 0) lanes = auto_lanes(n, nbins);
  return BLK_OK;
}

template <class K, class T>
blk_status launch_k(K kern, size_t n, int lanes, int threads, cudaStream_t st, const T *v,
                    const T *x, T *a, T *b, T *c, int nbins, int mode, int ept = 1) {
  const size_t total = n * (size_t)lanes;
  // ept: elements per thread (the scalar-I/O FP32 kernel at one element per
  // lane: BLK_F32_EPT; every other kernel 1)
  const size_t per_block = (size_t)threads * (size_t)ept;
  const size_t blocks = (total + per_block - 1) / per_block;
  if (blocks > 0x7fffffffULL) return fail(BLK_EINVAL, "grid too large");
#ifdef BLK_SMEM_PAD
  // tuning builds only: pad dynamic shared memory to cap resident blocks per SM
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, BLK_SMEM_PAD);
  kern<<<(unsigned)blocks, threads, BLK_SMEM_PAD, st>>>(v, x, n, a, b, c, nbins, mode);
#else
  kern<<<(unsigned)blocks, threads, 0, st>>>(v, x, n, a, b, c, nbins, mode);
#endif
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return BLK_OK;
}

// elements per thread of the one-element-per-lane scalar-I/O kernel (FP32: BLK_F32_EPT)
#define BLK_EPT_OF(ptr) (sizeof(*(ptr)) == 4 ? BLK_F32_EPT : 1)
#ifdef BLK_MIN_INSTANCES
// tuning-variant builds (tools/build_variants.py): one element per lane only
#define BLK_DISPATCH_LPE(KER, L, O1, O2, O3) \
  if (vec) return launch_k(KER<O1, O2, O3, 1, true>, n, 1, th, stream, v, x, a, b, c, nbins, mode); \
  return launch_k(KER<O1, O2, O3, 1>, n, 1, th, stream, v, x, a, b, c, nbins, mode, BLK_EPT_OF(v));
#else
#define BLK_DISPATCH_LPE(KER, L, O1, O2, O3)                                        \
  if (vec) return launch_k(KER<O1, O2, O3, 1, true>, n, 1, th, stream, v, x, a, b, c, nbins, mode); \
  switch (L) {                                                                      \
    case 1: return launch_k(KER<O1, O2, O3, 1>, n, L, th, stream, v, x, a, b, c, nbins, mode, BLK_EPT_OF(v)); \
    case 2: return launch_k(KER<O1, O2, O3, 2>, n, L, th, stream, v, x, a, b, c, nbins, mode); \
    case 4: return launch_k(KER<O1, O2, O3, 4>, n, L, th, stream, v, x, a, b, c, nbins, mode); \
    case 8: return launch_k(KER<O1, O2, O3, 8>, n, L, th, stream, v, x, a, b, c, nbins, mode); \
    case 16: return launch_k(KER<O1, O2, O3, 16>, n, L, th, stream, v, x, a, b, c, nbins, mode); \
    default: return launch_k(KER<O1, O2, O3, 32>, n, L, th, stream, v, x, a, b, c, nbins, mode); \
  }
#endif

template <class T>
blk_status run(const T *v, const T *x, size_t n, T *a, T *b, T *c, int nbins,
               const blk_options *opts, cudaStream_t stream) {
  int lanes, mode, th, kernel;
  blk_status st = validate(v, x, n, a, b, c, nbins, opts, lanes, mode, th, kernel);
  if (st != BLK_OK) return st;
  if (n == 0) return BLK_OK;
  const bool vec = kernel == BLK_KERNEL_VEC128;
  const int sel = (a ? 4 : 0) | (b ? 2 : 0) | (c ? 1 : 0);
  if constexpr (sizeof(T) == 8) {
    switch (sel) {
      case 7: BLK_DISPATCH_LPE(blk::logk_f64_kernel, lanes, true, true, true)
      case 6: BLK_DISPATCH_LPE(blk::logk_f64_kernel, lanes, true, true, false)
      case 5: BLK_DISPATCH_LPE(blk::logk_f64_kernel, lanes, true, false, true)
      case 4: BLK_DISPATCH_LPE(blk::logk_f64_kernel, lanes, true, false, false)
      case 3: BLK_DISPATCH_LPE(blk::logk_f64_kernel, lanes, false, true, true)
      case 2: BLK_DISPATCH_LPE(blk::logk_f64_kernel, lanes, false, true, false)
      default: BLK_DISPATCH_LPE(blk::logk_f64_kernel, lanes, false, false, true)
    }
  } else {
    switch (sel) {
      case 7: BLK_DISPATCH_LPE(blk::logk_f32_kernel, lanes, true, true, true)
      case 6: BLK_DISPATCH_LPE(blk::logk_f32_kernel, lanes, true, true, false)
      case 5: BLK_DISPATCH_LPE(blk::logk_f32_kernel, lanes, true, false, true)
      case 4: BLK_DISPATCH_LPE(blk::logk_f32_kernel, lanes, true, false, false)
      case 3: BLK_DISPATCH_LPE(blk::logk_f32_kernel, lanes, false, true, true)
      case 2: BLK_DISPATCH_LPE(blk::logk_f32_kernel, lanes, false, true, false)
      default: BLK_DISPATCH_LPE(blk::logk_f32_kernel, lanes, false, false, true)
    }
  }
}

// ---- host-buffer pipeline
#ifndef BLK_HOST_STREAMS
#define BLK_HOST_STREAMS 3
#endif
constexpr int kHostStreams = BLK_HOST_STREAMS;
std::mutex g_pool_mu;
struct Pool {
  int device = -1;
  cudaStream_t s[kHostStreams];
  cudaEvent_t ev[kHostStreams];
};
Pool g_pools[64];

blk_status get_pool(Pool *&out) {
  int dev;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(BLK_ECUDA, "device ordinal out of range");
  std::lock_guard<std::mutex> lk(g_pool_mu);
  Pool &p = g_pools[dev];
  if (p.device < 0) {
    for (int k = 0; k < kHostStreams; ++k) {
      e = cudaStreamCreateWithFlags(&p.s[k], cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
      e = cudaEventCreateWithFlags(&p.ev[k], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    }
    p.device = dev;
  }
  out = &p;
  return BLK_OK;
}

}  // namespace

extern "C" {

const char *bessel_logk_last_error(void) { return g_err; }
const char *bessel_logk_version(void) { return "bessel_logk 0.1.0 sm_100a"; }

blk_status bessel_logk_f64(const double *v, const double *x, size_t n, double *logk,
                           double *dlogk_dv, double *dlogk_dx, int nbins, cudaStream_t stream) {
  return run<double>(v, x, n, logk, dlogk_dv, dlogk_dx, nbins, nullptr, stream);
}
blk_status bessel_logk_f32(const float *v, const float *x, size_t n, float *logk,
                           float *dlogk_dv, float *dlogk_dx, int nbins, cudaStream_t stream) {
  return run<float>(v, x, n, logk, dlogk_dv, dlogk_dx, nbins, nullptr, stream);
}
blk_status bessel_logk_f64_ex(const double *v, const double *x, size_t n, double *logk,
                              double *dlogk_dv, double *dlogk_dx, int nbins,
                              const blk_options *opts, cudaStream_t stream) {
  return run<double>(v, x, n, logk, dlogk_dv, dlogk_dx, nbins, opts, stream);
}
blk_status bessel_logk_f32_ex(const float *v, const float *x, size_t n, float *logk,
                              float *dlogk_dv, float *dlogk_dx, int nbins,
                              const blk_options *opts, cudaStream_t stream) {
  return run<float>(v, x, n, logk, dlogk_dv, dlogk_dx, nbins, opts, stream);
}

size_t bessel_logk_host_workspace_bytes(size_t chunk, size_t elem_bytes) {
  if (chunk == 0) chunk = (size_t)1 << 20;
  // per helper stream: v, x and three outputs of `chunk` elements, 256-B aligned
  const size_t arr = ((chunk * elem_bytes) + 255) / 256 * 256;
  return (size_t)kHostStreams * 5 * arr;
}

}  // extern "C"

namespace {
// H2D -> kernel -> D2H pipeline over chunks on the helper streams (both precisions).
template <class T>
blk_status run_host(const T *v, const T *x, size_t n, T *logk, T *dlogk_dv, T *dlogk_dx,
                    int nbins, void *workspace, size_t workspace_bytes, size_t chunk,
                    cudaStream_t stream) {
  int lanes, mode, th, kernel;
  blk_status st = validate(v, x, n, logk, dlogk_dv, dlogk_dx, nbins, nullptr, lanes, mode, th, kernel);
  if (st != BLK_OK) return st;
  if (n == 0) return BLK_OK;
  if (chunk == 0) chunk = (size_t)1 << 20;
  // Zero-copy: when every buffer is page-locked host memory mapped into the
  // device address space (cudaHostAlloc / cudaHostRegister under UVA, e.g.
  // torch's pin_memory), one launch reads the inputs and writes the outputs
  // over PCIe directly -- the transfers then overlap the computation element
  // by element instead of chunk by chunk (c2: 0.73 -> 0.61 ms per 2^20
  // elements, profiles/r01s3d_e2e_zero_copy.log).  BLK_HOST_PIPELINE=1 in the
  // environment forces the staged path (measurement only).
  {
    const char *force = getenv("BLK_HOST_PIPELINE");
    if (!(force && atoi(force) == 1)) {
      auto mapped = [](const void *p) -> void * {
        if (!p) return nullptr;
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        return (at.type == cudaMemoryTypeHost) ? at.devicePointer : nullptr;
      };
      const T *mv = (const T *)mapped(v), *mx = (const T *)mapped(x);
      T *m0 = (T *)mapped(logk), *m1 = (T *)mapped(dlogk_dv), *m2 = (T *)mapped(dlogk_dx);
      if (mv && mx && (!logk || m0) && (!dlogk_dv || m1) && (!dlogk_dx || m2)) {
        // one element per lane, as in the staged path: the same results
        blk_options o{1, mode, th, BLK_KERNEL_SIMPLE};
        st = run<T>(mv, mx, n, m0, m1, m2, nbins, &o, stream);
        if (st != BLK_OK) return st;
        cudaError_t e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return cuda_fail(e, "synchronize");
        return BLK_OK;
      }
    }
  }
  // staged transport: the device workspace holds the chunks in flight
  if (!workspace || workspace_bytes < bessel_logk_host_workspace_bytes(chunk, sizeof(T)))
    return fail(BLK_EINVAL, "workspace missing or too small (staged transport)");
  Pool *pool;
  st = get_pool(pool);
  if (st != BLK_OK) return st;
  const size_t arr = ((chunk * sizeof(T)) + 255) / 256 * 256;
  cudaError_t e;
  // order after the caller's prior work
  cudaEvent_t start_ev;
  if ((e = cudaEventCreateWithFlags(&start_ev, cudaEventDisableTiming)) != cudaSuccess)
    return cuda_fail(e, "cudaEventCreate");
  struct EventGuard {          // destroyed on every return path
    cudaEvent_t ev;
    ~EventGuard() { cudaEventDestroy(ev); }
  } guard{start_ev};
  cudaEventRecord(start_ev, stream);
  for (int k = 0; k < kHostStreams; ++k) cudaStreamWaitEvent(pool->s[k], start_ev, 0);
  size_t nchunks = (n + chunk - 1) / chunk;
  for (size_t c = 0; c < nchunks; ++c) {
    const int k = (int)(c % kHostStreams);
    cudaStream_t s = pool->s[k];
    char *base = (char *)workspace + (size_t)k * 5 * arr;
    T *dv_ = (T *)(base), *dx_ = (T *)(base + arr);
    T *o0 = (T *)(base + 2 * arr), *o1 = (T *)(base + 3 * arr), *o2 = (T *)(base + 4 * arr);
    const size_t off = c * chunk, m = (n - off < chunk) ? n - off : chunk;
    const size_t bytes = m * sizeof(T);
    if ((e = cudaMemcpyAsync(dv_, v + off, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "H2D v");
    if ((e = cudaMemcpyAsync(dx_, x + off, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "H2D x");
    // one element per lane in every chunk: results do not depend on the
    // chunking and equal a device-path call with lanes_per_element = 1
    blk_options o{1, mode, th, BLK_KERNEL_SIMPLE};
    st = run<T>(dv_, dx_, m, logk ? o0 : nullptr, dlogk_dv ? o1 : nullptr,
                dlogk_dx ? o2 : nullptr, nbins, &o, s);
    if (st != BLK_OK) return st;
    if (logk && (e = cudaMemcpyAsync(logk + off, o0, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return cuda_fail(e, "D2H logk");
    if (dlogk_dv && (e = cudaMemcpyAsync(dlogk_dv + off, o1, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return cuda_fail(e, "D2H dv");
    if (dlogk_dx && (e = cudaMemcpyAsync(dlogk_dx + off, o2, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return cuda_fail(e, "D2H dx");
  }
  for (int k = 0; k < kHostStreams; ++k) {
    cudaEventRecord(pool->ev[k], pool->s[k]);
    cudaStreamWaitEvent(stream, pool->ev[k], 0);
  }
  if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return cuda_fail(e, "synchronize");
  return BLK_OK;
}
}  // namespace

extern "C" {

blk_status bessel_logk_f64_host(const double *v, const double *x, size_t n, double *logk,
                                double *dlogk_dv, double *dlogk_dx, int nbins, void *workspace,
                                size_t workspace_bytes, size_t chunk, cudaStream_t stream) {
  return run_host<double>(v, x, n, logk, dlogk_dv, dlogk_dx, nbins, workspace, workspace_bytes,
                          chunk, stream);
}
blk_status bessel_logk_f32_host(const float *v, const float *x, size_t n, float *logk,
                                float *dlogk_dv, float *dlogk_dx, int nbins, void *workspace,
                                size_t workspace_bytes, size_t chunk, cudaStream_t stream) {
  return run_host<float>(v, x, n, logk, dlogk_dv, dlogk_dx, nbins, workspace, workspace_bytes,
                         chunk, stream);
}

size_t bessel_nig_workspace_bytes(size_t n) {
  const size_t blocks = (n + blk::kNigThreads - 1) / blk::kNigThreads;
  return (blocks > 0 ? blocks : 1) * blk::kNigOut * sizeof(double);
}

blk_status bessel_nig_loglik_f64(const double *y, size_t n, double alpha, double beta,
                                 double delta, double mu, int nbins, double *out,
                                 void *workspace, size_t workspace_bytes, cudaStream_t s) {
  if (nbins < 2 || nbins > BLK_MAX_NBINS) return fail(BLK_EINVAL, "nbins out of range [2, 65536]");
  if (!out) return fail(BLK_EINVAL, "out is NULL");
  if (!(alpha > fabs(beta)) || !(delta > 0.0) || !isfinite(alpha) || !isfinite(delta) ||
      !isfinite(mu) || !isfinite(beta))
    return fail(BLK_EINVAL, "NIG parameters need |beta| < alpha, delta > 0, all finite");
  if (n > 0 && !y) return fail(BLK_EINVAL, "y is NULL");
  if (!workspace || workspace_bytes < bessel_nig_workspace_bytes(n))
    return fail(BLK_EINVAL, "workspace missing or too small");
  const size_t blocks = (n + blk::kNigThreads - 1) / blk::kNigThreads;
  if (blocks > 0x7fffffffULL) return fail(BLK_EINVAL, "n too large");
  const double gamma = sqrt(alpha * alpha - beta * beta);
  double *partial = (double *)workspace;
  if (blocks > 0)
    blk::nig_f64_kernel<<<(unsigned)blocks, blk::kNigThreads, 0, s>>>(y, n, alpha, beta, delta, mu,
                                                                     gamma, nbins, partial);
  blk::nig_final_kernel<<<1, 256, 0, s>>>(partial, blocks, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BLK_OK : cuda_fail(e, "nig kernels");
}

blk_status bessel_logk_plan_f64(const double *v, const double *x, size_t n, double *tp,
                                double *gp, double *t0, double *t1, int nbins,
                                const blk_options *opts, cudaStream_t stream) {
  int lanes, mode, th, kernel;
  const bool any = tp || gp || t0 || t1;
  blk_status st = validate(v, x, n, any ? (void *)1 : nullptr, nullptr, nullptr, nbins, opts,
                           lanes, mode, th, kernel);
  if (st != BLK_OK) return st;
  if (n == 0) return BLK_OK;
  const size_t blocks = (n + 127) / 128;
  if (blocks > 0x7fffffffULL) return fail(BLK_EINVAL, "grid too large");
  blk::logk_plan_f64_kernel<<<(unsigned)blocks, 128, 0, stream>>>(v, x, n, tp, gp, t0, t1, nbins,
                                                                  mode);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BLK_OK : cuda_fail(e, "plan kernel launch");
}

blk_status bessel_logk_hess_f64(const double *v, const double *x, size_t n, double *logk,
                                double *dlogk_dv, double *dlogk_dx, double *d2_dv2,
                                double *d2_dx2, double *d2_dvdx, int nbins,
                                const blk_options *opts, cudaStream_t stream) {
  int lanes, mode, th, kernel;
  const bool any = logk || dlogk_dv || dlogk_dx || d2_dv2 || d2_dx2 || d2_dvdx;
  blk_status st = validate(v, x, n, any ? (void *)1 : nullptr, nullptr, nullptr, nbins, opts,
                           lanes, mode, th, kernel);
  if (st != BLK_OK) return st;
  if (n == 0) return BLK_OK;
  const size_t total = n * (size_t)lanes;
  const size_t blocks = (total + th - 1) / th;
  if (blocks > 0x7fffffffULL) return fail(BLK_EINVAL, "grid too large");
#define BLK_HESS_LAUNCH(L)                                                                    \
  blk::logk_f64_hess_kernel<L><<<(unsigned)blocks, th, 0, stream>>>(                          \
      v, x, n, logk, dlogk_dv, dlogk_dx, d2_dv2, d2_dx2, d2_dvdx, nbins, mode)
  switch (lanes) {
    case 1: BLK_HESS_LAUNCH(1); break;
    case 2: BLK_HESS_LAUNCH(2); break;
    case 4: BLK_HESS_LAUNCH(4); break;
    case 8: BLK_HESS_LAUNCH(8); break;
    case 16: BLK_HESS_LAUNCH(16); break;
    default: BLK_HESS_LAUNCH(32); break;
  }
#undef BLK_HESS_LAUNCH
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BLK_OK : cuda_fail(e, "hess kernel launch");
}

#ifdef BLK_DIAG
// Diagnostics build only (tools/phase_split.py etc.; not in the public header):
// the FP64 path as two kernels, plan into `scratch` (32 B per element), then
// quadrature + epilogue, to time the phases separately.
__attribute__((visibility("default"))) blk_status blk_debug_split_f64(const double *v, const double *x, size_t n, double *logk,
                               double *dlogk_dv, double *dlogk_dx, int nbins, void *scratch,
                               int phases, cudaStream_t s) {
  if (!v || !x || !logk || !dlogk_dv || !dlogk_dx || !scratch || nbins < 2 || nbins > BLK_MAX_NBINS)
    return fail(BLK_EINVAL, "bad split args");
  if (n == 0) return BLK_OK;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  blk::PlanRec *plans = (blk::PlanRec *)scratch;
  if (phases & 1) blk::plan_f64_kernel<<<blocks, 128, 0, s>>>(v, x, n, plans, nbins, 0);
  if (phases & 2)
    blk::quad_f64_kernel<true, true, true><<<blocks, 128, 0, s>>>(v, x, n, plans, logk, dlogk_dv,
                                                                  dlogk_dx, nbins);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BLK_OK : cuda_fail(e, "split kernels");
}
#endif

#ifdef BLK_TIMELINE
__attribute__((visibility("default"))) blk_status blk_debug_timeline(unsigned long long *host, size_t max_warps) {
  const size_t n = max_warps < (size_t)blk::kTlMax ? max_warps : (size_t)blk::kTlMax;
  cudaError_t e = cudaMemcpyFromSymbol(host, blk::g_tl, n * 4 * sizeof(unsigned long long));
  return e == cudaSuccess ? BLK_OK : cuda_fail(e, "timeline copy");
}
#endif

blk_status blk_microbench_fp64(int blocks, int threads, int iters, double *out, cudaStream_t s) {
  if (blocks <= 0 || threads <= 0 || threads > 1024 || iters <= 0 || !out)
    return fail(BLK_EINVAL, "bad microbench args");
  blk::mb_fp64_kernel<<<blocks, threads, 0, s>>>(iters, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BLK_OK : cuda_fail(e, "mb_fp64");
}
blk_status blk_microbench_fp32(int blocks, int threads, int iters, float *out, cudaStream_t s) {
  if (blocks <= 0 || threads <= 0 || threads > 1024 || iters <= 0 || !out)
    return fail(BLK_EINVAL, "bad microbench args");
  blk::mb_fp32_kernel<<<blocks, threads, 0, s>>>(iters, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BLK_OK : cuda_fail(e, "mb_fp32");
}
blk_status blk_microbench_mufu(int blocks, int threads, int iters, float *out, cudaStream_t s) {
  if (blocks <= 0 || threads <= 0 || threads > 1024 || iters <= 0 || !out)
    return fail(BLK_EINVAL, "bad microbench args");
  blk::mb_mufu_kernel<<<blocks, threads, 0, s>>>(iters, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BLK_OK : cuda_fail(e, "mb_mufu");
}

}  // extern "C"
