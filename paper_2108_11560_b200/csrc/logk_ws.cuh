// logk_ws.cuh -- warp-specialized persistent FP64 kernel.
//
// The hot path has two phases with disjoint hardware needs: range finding
// (Alg. 1-3 lines 2-9, FP32 FMA pipe + MUFU, latency-bound dependent chains)
// and the fixed-bin quadrature (Eq. (int) + Sec. 4.1 sums, FP64 pipe).  In
// the one-element-per-thread kernel every warp alternates between them, so
// the FP64 pipe idles whenever the resident warps happen to be range-finding.
// Here each CTA splits its warps by role:
//   producer warps : load v, x for a tile of 32 elements, find the plan
//                    (t0, h, shift) and publish it in a shared-memory ring;
//   consumer warps : take a plan, run the quadrature (FP64) and the epilogue,
//                    store the outputs.
// The ring has kSlots slots guarded by mbarriers (full: 32 producer lanes
// arrive; empty: 32 consumer lanes arrive).  CTAs are persistent: CTA b owns
// tiles b, b + G, b + 2G, ...; within a CTA producers and consumers claim
// local tiles in increasing order through shared counters, so the ring is
// filled and drained in order.  Results are bit-identical to the simple
// kernel (same per-element code, same order of operations).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "logk_quad.cuh"
#include "logk_range.cuh"

namespace blk {

#ifndef BLK_WS_NP
#define BLK_WS_NP 4
#endif
#ifndef BLK_WS_NC
#define BLK_WS_NC 12
#endif
#ifndef BLK_WS_MINB
#define BLK_WS_MINB 1
#endif
constexpr int kWsProducers = BLK_WS_NP;   // warps
constexpr int kWsConsumers = BLK_WS_NC;   // warps
constexpr int kWsThreads = 32 * (kWsProducers + kWsConsumers);
constexpr int kSlots = 16;

struct SlotLane {
  double t0, h, gp, v, x;
  int flags;   // bit0 ok, bit1 clamp, bit2 v negative
  int pad;
};

struct WsShared {
  SlotLane slot[kSlots][32];
  unsigned long long full[kSlots];
  unsigned long long empty[kSlots];
  int prod_next, cons_next;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <bool LOGK, bool DV, bool DX>
__global__ void __launch_bounds__(kWsThreads, BLK_WS_MINB)
logk_f64_ws_kernel(const double *__restrict__ vin, const double *__restrict__ xin, size_t n_el,
                   double *__restrict__ logk, double *__restrict__ dlogk_dv,
                   double *__restrict__ dlogk_dx, int nbins, int range_mode) {
  extern __shared__ __align__(16) unsigned char ws_raw[];
  WsShared &S = *reinterpret_cast<WsShared *>(ws_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  load_exp_table();
  if (threadIdx.x < kSlots) {
    mbar_init(&S.full[threadIdx.x], 32);
    mbar_init(&S.empty[threadIdx.x], 32);
  }
  if (threadIdx.x == 0) { S.prod_next = 0; S.cons_next = 0; }
  __syncthreads();

  const size_t n_tiles = (n_el + 31) / 32;
  const size_t G = gridDim.x, b = blockIdx.x;
  const size_t my_tiles = (b < n_tiles) ? (n_tiles - b + G - 1) / G : 0;

  if (warp < kWsProducers) {
    // ------------------------------------------------------------ producer
    for (;;) {
      int j = 0;
      if (lane == 0) j = atomicAdd(&S.prod_next, 1);
      j = __shfl_sync(0xffffffffu, j, 0);
      if ((size_t)j >= my_tiles) break;
      const int s = j % kSlots;
      if (j >= kSlots) mbar_wait(&S.empty[s], ((j / kSlots) - 1) & 1);
      const size_t i = (b + (size_t)j * G) * 32 + lane;
      const bool live = i < n_el;
      const double vraw = live ? vin[i] : 1.0;
      const double x = live ? xin[i] : 1.0;
      const bool valid = live && (x > 0.0) && isfinite(x) && isfinite(vraw);
      const double v = fabs(vraw);
      double t0 = 0.0, t1 = 0.0, gp = 0.0, dmin = 0.0;
      bool ok = false;
      if (valid) {
        if (range_mode == BLK_RANGE_AUTO && f32_plan_domain(v, x)) {
          const Plan<float> p = make_plan_f32(v, x, kLogEpsF64, fz_tol_for(nbins));
          ok = p.ok; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
        } else {
          const Plan<double> p = make_plan_f64_tab(v, x, kLogEpsF64);
          ok = p.ok; t0 = p.t0; t1 = p.t1; gp = p.gp; dmin = p.dmin;
        }
        ok = ok && isfinite(t1) && isfinite(gp) && t1 > t0;
      }
      SlotLane &sl = S.slot[s][lane];
      sl.t0 = t0;
      sl.h = (t1 - t0) * rcp64((double)nbins);
      sl.gp = gp;
      sl.v = v;
      sl.x = x;
      sl.flags = (ok ? 1 : 0) | (dmin > -600.0 ? 0 : 2) | (vraw < 0.0 ? 4 : 0);
      mbar_arrive(&S.full[s]);
    }
  } else {
    // ------------------------------------------------------------ consumer
    for (;;) {
      int j = 0;
      if (lane == 0) j = atomicAdd(&S.cons_next, 1);
      j = __shfl_sync(0xffffffffu, j, 0);
      if ((size_t)j >= my_tiles) break;
      const int s = j % kSlots;
      mbar_wait(&S.full[s], (j / kSlots) & 1);
      const SlotLane sl = S.slot[s][lane];
      mbar_arrive(&S.empty[s]);
      const size_t i = (b + (size_t)j * G) * 32 + lane;
      const bool ok = sl.flags & 1;
      Sums64 r{0.0, 0.0, 0.0};
      if (ok) {
        if (!(sl.flags & 2))
          r = quad_f64<DV, DX, false>(sl.v, sl.x, sl.t0, sl.h, sl.gp, nbins, 0, nbins + 1, g_exp_tab);
        else
          r = quad_f64<DV, DX, true>(sl.v, sl.x, sl.t0, sl.h, sl.gp, nbins, 0, nbins + 1, g_exp_tab);
      }
      if (i < n_el) {
        const double nanv = __longlong_as_double(0x7ff8000000000000ULL);
        const double rc = rcp64(r.S0);
        const double sgn = (sl.flags & 4) ? -1.0 : 1.0;
        if (LOGK) logk[i] = ok ? sl.gp + log_sum(sl.h * r.S0) : nanv;
        if (DV) dlogk_dv[i] = ok ? sgn * (r.S1 * rc) : nanv;
        if (DX) dlogk_dx[i] = ok ? -(r.S2 * rc) : nanv;
      }
    }
  }
}

}  // namespace blk
