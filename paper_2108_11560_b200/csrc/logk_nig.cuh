// logk_nig.cuh -- fused normal-inverse-Gaussian log-likelihood and gradient
// (the motivating application).
//
//   log p(y) = log a + log d - log pi + d g + b (y - m) - log q + log K_1(a q),
//   q = sqrt(d^2 + (y - m)^2),  g = sqrt(a^2 - b^2)   (a = alpha, b = beta,
//   d = delta, m = mu; |b| < a, d > 0)
//
// Each thread evaluates log K_1(z) and dlogK_1/dz at z = a q with the same
// plan + fixed-bin quadrature as the batched kernel (v = 1, no dv sum), forms
// log p and its gradient in (a, b, d, m):
//   d/da = 1/a + d a/g + q D,   d/db = (y - m) - d b/g,
//   d/dd = 1/d + g - d/q^2 + a D d/q,   d/dm = -b + (y - m)/q^2 - a D (y - m)/q,
// with D = dlogK_1/dz, and the block reduces the five sums in a fixed order
// (warp shuffles, then shared memory).  A one-block second kernel reduces the
// per-block partials in a fixed order, so the result is deterministic.  The
// cross-GPU sum is one NCCL all_reduce of these five numbers (dist.py).
#pragma once
#include <cuda_runtime.h>

#include "logk_quad.cuh"
#include "logk_range.cuh"

#ifndef BLK_SMART_NIG
#define BLK_SMART_NIG true
#endif

namespace blk {

constexpr int kNigThreads = 128;
constexpr int kNigOut = 5;

__device__ __forceinline__ double warp_sum(double a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

__global__ void __launch_bounds__(kNigThreads, BLK_MINB)
nig_f64_kernel(const double *__restrict__ y, size_t n, double a, double b, double d, double m,
               double g, int nbins, double *__restrict__ partial) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double yi = i < n ? y[i] : 0.0;   // issued ahead of the table copy
  load_exp_table_sync();
  __shared__ double red[kNigOut][kNigThreads / 32];
  double c[kNigOut] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (i < n) {
    const double r = yi - m;
    const double q2 = fma(r, r, d * d), q = sqrt(q2);
    const double z = a * q;
    double lk = __longlong_as_double(0x7ff8000000000000ULL), D = lk;
    if (z > 0.0 && isfinite(z)) {
      double t0, t1, gp, dmin;
      bool ok;
      if (use_f32_plan(0, nbins, 1.0, z)) {
        const Plan<float> p = make_plan_f32<BLK_SMART_NIG>(1.0, z, kLogEpsF64, fz_tol_for(nbins));
        ok = p.ok; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
      } else {
        const Plan<double> p = make_plan_f64_tab(1.0, z, kLogEpsF64);
        ok = p.ok; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
      }
      ok = ok && isfinite(t1) && isfinite(gp) && t1 > t0 && t1 < kTMax;   // R23
      if (ok) {
        const double h = (t1 - t0) * rcp64((double)nbins);
        const Sums64 s = dmin > -600.0
                             ? quad_f64<false, true, false>(1.0, z, t0, h, gp, nbins, 0, nbins + 1, g_exp_tab)
                             : quad_f64<false, true, true>(1.0, z, t0, h, gp, nbins, 0, nbins + 1, g_exp_tab);
        const double rs = rcp64(s.S0);
        lk = gp + log_sum(h * s.S0);
        D = -(s.S2 * rs);
      }
    }
    const double iq = rcp64(q), iq2 = iq * iq;
    c[0] = log(a * d * iq) - 1.1447298858494002 + d * g + b * r + lk;   // log pi
    c[1] = 1.0 / a + d * a / g + q * D;
    c[2] = r - d * b / g;
    c[3] = 1.0 / d + g - d * iq2 + a * D * d * iq;
    c[4] = -b + r * iq2 - a * D * r * iq;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kNigOut; ++k) {
    const double w = warp_sum(c[k]);
    if (lane == 0) red[k][warp] = w;
  }
  __syncthreads();
  if (threadIdx.x < kNigOut) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < kNigThreads / 32; ++w) acc += red[threadIdx.x][w];
    partial[(size_t)blockIdx.x * kNigOut + threadIdx.x] = acc;
  }
}

// Fixed-order reduction of nblocks x 5 partials by one block of 256 threads.
__global__ void __launch_bounds__(256)
nig_final_kernel(const double *__restrict__ partial, size_t nblocks, double *__restrict__ out) {
  __shared__ double red[kNigOut][256 / 32];
  double acc[kNigOut] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (size_t j = threadIdx.x; j < nblocks; j += blockDim.x) {
#pragma unroll
    for (int k = 0; k < kNigOut; ++k) acc[k] += partial[j * kNigOut + k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kNigOut; ++k) {
    const double w = warp_sum(acc[k]);
    if (lane == 0) red[k][warp] = w;
  }
  __syncthreads();
  if (threadIdx.x < kNigOut) {
    double s = 0.0;
    for (int w = 0; w < 256 / 32; ++w) s += red[threadIdx.x][w];
    out[threadIdx.x] = s;
  }
}

}  // namespace blk
