// logk_io.cuh -- warp-cooperative 128-bit loads and stores of the v / x /
// output streams (BASELINE.json north_star (3): "vectorised, coalesced
// 128-bit loads and stores of the v/x/output streams").
//
// With one element per lane, a warp owns 32 consecutive elements: 256 B of
// each FP64 stream (128 B FP32).  Instead of one 8-B (4-B) load per lane and
// stream, the warp moves whole 16-B vectors: FP64, lanes 0-15 load v and lanes
// 16-31 load x (one LDG.128 per lane); FP32, lanes 0-7 load v and 8-15 load x.
// The vectors are transposed to one element per lane through a warp-private
// slice of shared memory (STS.128, __syncwarp, LDS), and the outputs go back
// the same way (STS per lane and output, LDS.128, STG.128).  Used by the
// kernels' VEC instantiations (BLK_KERNEL_VEC128; the host checks that every
// stream is 16-B aligned) for warps whose 32 elements are all in range; the
// ragged last warp takes the scalar path.  Results are identical to the scalar
// kernels' (the arithmetic does not depend on how an element was loaded).
// Not the default: at ~3% of HBM bandwidth the kernels gain nothing from
// wider accesses, and the transposes cost 0.8% (FP64, c3) / 1.7% (FP32, c4)
// on B200 (profiles/r02io_vec128_ab.log).
#pragma once
#include <cuda_runtime.h>

namespace blk {

// Shared staging: each warp uses its own slice of kIoPerWarp values (3 per
// lane: the outputs; the inputs use the first 64).  Everything is derived
// from the element index i (= the global thread index with one element per
// lane) so that nothing but i stays live across the computation: lane = i % 32,
// the warp's first element w0 = i - lane, and its slice (i / 32) % 4 -- the
// at most 4 warps of a block (<= 128 threads) have consecutive i / 32.
constexpr int kIoPerWarp = 3 * 32;
constexpr int kIoWarps = 4;

template <class T>
struct Vec16;
template <>
struct Vec16<double> { using type = double2; static constexpr int n = 2; };
template <>
struct Vec16<float> { using type = float4; static constexpr int n = 4; };

// Step 1 (before any barrier, so its latency overlaps the caller's setup):
// lane L issues one 16-B load, of v for L in [0, 32/V), of x for
// [32/V, 64/V) and nothing above (V = values per vector: 2 FP64, 4 FP32).
template <class T>
__device__ __forceinline__ typename Vec16<T>::type io_load_issue(const T *__restrict__ vin,
                                                                 const T *__restrict__ xin,
                                                                 size_t i) {
  using V = typename Vec16<T>::type;
  const int lane = (int)(i & 31);
  const size_t w0 = i - lane;
  constexpr int lpa = 32 / Vec16<T>::n;   // lanes per array: 16 (FP64) / 8 (FP32)
  V r{};
  if (lane < 2 * lpa) {
    const T *src = (lane < lpa) ? vin : xin;
    r = __ldg(reinterpret_cast<const V *>(src + w0) + (lane % lpa));
  }
  return r;
}

// Step 2: transpose through the warp's slice of s_io: lane L gets element
// w0 + L's v and x.
template <class T>
__device__ __forceinline__ void io_load_finish(T *s_io, typename Vec16<T>::type r, size_t i,
                                               T &v, T &x) {
  using V = typename Vec16<T>::type;
  const int lane = (int)(i & 31);
  T *sw = s_io + ((i >> 5) % kIoWarps) * kIoPerWarp;
  constexpr int lpa = 32 / Vec16<T>::n;
  if (lane < 2 * lpa) reinterpret_cast<V *>(sw)[lane] = r;   // sw[0,32) = v, sw[32,64) = x
  __syncwarp();
  v = sw[lane];
  x = sw[32 + lane];
}

// The outputs of the warp's 32 elements, present ones only (compile-time
// flags), compacted in the order logk, dv, dx: each lane writes its values to
// sw, then lane q stores 16-B vector q of the compacted [K][32] block.
template <class T, bool A, bool B, bool C, bool WAR_SYNC = true>
__device__ __forceinline__ void io_store(T *s_io, size_t i, T a, T b, T c,
                                         T *__restrict__ pa, T *__restrict__ pb,
                                         T *__restrict__ pc) {
  using V = typename Vec16<T>::type;
  const int lane = (int)(i & 31);
  const size_t w0 = i - lane;
  T *sw = s_io + ((i >> 5) % kIoWarps) * kIoPerWarp;
  constexpr int K = int(A) + int(B) + int(C);
  if (K == 0) return;
  constexpr int lpa = 32 / Vec16<T>::n;
  T *const o0 = A ? pa : (B ? pb : pc), *const o1 = (A && B) ? pb : pc, *const o2 = pc;
  if (WAR_SYNC) __syncwarp();   // every lane has read its inputs from sw
  int k = 0;
  if (A) sw[32 * (k++) + lane] = a;
  if (B) sw[32 * (k++) + lane] = b;
  if (C) sw[32 * (k++) + lane] = c;
  __syncwarp();
#pragma unroll
  for (int q = lane; q < K * lpa; q += 32) {
    const int j = q / lpa;
    T *o = (j == 0) ? o0 : ((j == 1) ? o1 : o2);
    reinterpret_cast<V *>(o + w0)[q % lpa] = reinterpret_cast<const V *>(sw)[q];
  }
}

}  // namespace blk
