// logk_split.cuh -- DIAGNOSTICS BUILD ONLY (-DBLK_DIAG, tools/): the hot path
// as two kernels (plan, then quadrature) with the per-element plan in a
// caller-provided scratch array, to time the two phases separately
// (blk_debug_split_f64).  Same range finders as the fused kernel (FP32, or the
// table-exp FP64 one outside the FP32 domain), so results equal it bit for bit.
#pragma once
#include <cuda_runtime.h>

#include "logk_quad.cuh"
#include "logk_range.cuh"

namespace blk {

struct PlanRec {
  double t0, h, gp;
  int flags;   // bit0 ok, bit1 clamp, bit2 v negative
  int pad;
};

__global__ void __launch_bounds__(128)
plan_f64_kernel(const double *__restrict__ vin, const double *__restrict__ xin, size_t n_el,
                PlanRec *__restrict__ plans, int nbins, int range_mode) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  load_exp_table_sync();   // for make_plan_f64_tab, before any thread leaves
  if (i >= n_el) return;
  const double vraw = vin[i], x = xin[i];
  const bool valid = (x > 0.0) && isfinite(x) && isfinite(vraw);
  const double v = fabs(vraw);
  double t0 = 0.0, t1 = 0.0, gp = 0.0, dmin = 0.0;
  bool ok = false;
  if (valid) {
    if (use_f32_plan(range_mode, nbins, v, x)) {
      const Plan<float> p = make_plan_f32(v, x, kLogEpsF64, fz_tol_for(nbins));
      ok = p.ok; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
    } else {
      const Plan<double> p = make_plan_f64_tab(v, x, kLogEpsF64);
      ok = p.ok; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
    }
    ok = ok && isfinite(t1) && isfinite(gp) && t1 > t0 && t1 < kTMax;   // as element_plan_f64 (R23)
  }
  PlanRec r;
  r.t0 = t0; r.h = (t1 - t0) * rcp64((double)nbins); r.gp = gp;
  r.flags = (ok ? 1 : 0) | (dmin > -600.0 ? 0 : 2) | (vraw < 0.0 ? 4 : 0);
  r.pad = 0;
  plans[i] = r;
}

template <bool LOGK, bool DV, bool DX>
__global__ void __launch_bounds__(128, BLK_MINB)
quad_f64_kernel(const double *__restrict__ vin, const double *__restrict__ xin, size_t n_el,
                const PlanRec *__restrict__ plans, double *__restrict__ logk,
                double *__restrict__ dlogk_dv, double *__restrict__ dlogk_dx, int nbins) {
  load_exp_table_sync();
  const double *tab = g_exp_tab;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_el) return;
  const PlanRec pl = plans[i];
  const double v = fabs(vin[i]), x = xin[i];
  const bool ok = pl.flags & 1;
  Sums64 r{0.0, 0.0, 0.0};
  if (ok) {
    if (!(pl.flags & 2)) r = quad_f64<DV, DX, false>(v, x, pl.t0, pl.h, pl.gp, nbins, 0, nbins + 1, tab);
    else r = quad_f64<DV, DX, true>(v, x, pl.t0, pl.h, pl.gp, nbins, 0, nbins + 1, tab);
  }
  const double nanv = __longlong_as_double(0x7ff8000000000000ULL);
  const double rc = rcp64(r.S0);
  const double sgn = (pl.flags & 4) ? -1.0 : 1.0;
  if (LOGK) logk[i] = ok ? pl.gp + log_sum(pl.h * r.S0) : nanv;
  if (DV) dlogk_dv[i] = ok ? sgn * (r.S1 * rc) : nanv;
  if (DX) dlogk_dx[i] = ok ? -(r.S2 * rc) : nanv;
}

}  // namespace blk
