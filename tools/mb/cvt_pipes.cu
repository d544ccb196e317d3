// Which pipe runs FRND.F64 (cvt.rni.f64.f64) and F2I.F64 (cvt.rni.s32.f64) on
// sm_100a, and at what rate?  Question behind it: can the exp reduction of the
// FP64 node loop (k = rint(a'), r' = a' - k) move two of its three FP64
// instructions to another pipe?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cvt_pipes cvt_pipes.cu
// Each kernel: 8 independent streams per thread, inputs varied per iteration
// by an integer add (ALU pipe), results folded with LOP3 (ALU pipe), so the
// measured rate is that of the instruction under test.  Reported as warp-level
// instructions per clock per SM at 1.965 GHz.  Result on B200
// (profiles/r02zs_cvt_pipes.log; ncu: sm__inst_executed_pipe_xu counts them):
// FRND.F64 and F2I.F64 run on the XU at ~16 lanes/clk/SM like MUFU.EX2 and
// share it with MUFU and with each other; next to DFMA they overlap.
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
#define UNR 4

__device__ __forceinline__ double frnd(double a) {
  double r;
  asm volatile("cvt.rni.f64.f64 %0, %1;" : "=d"(r) : "d"(a));
  return r;
}
__device__ __forceinline__ int f2i(double a) {
  int r;
  asm volatile("cvt.rni.s32.f64 %0, %1;" : "=r"(r) : "d"(a));
  return r;
}
__device__ __forceinline__ float ex2(float a) {
  float r;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ double bump(double a, int i) {   // integer-only change of the input
  return __hiloint2double(__double2hiint(a), __double2loint(a) + i);
}

// MODE bits: 1 FRND, 2 F2I, 4 DFMA, 8 MUFU.EX2
template <int MODE>
__global__ void k(int iters, unsigned *out, long long *clk) {
  double a[CH], d[CH];
  float f[CH];
  for (int j = 0; j < CH; ++j) {
    a[j] = 1000.25 + j + threadIdx.x * 1e-3;
    d[j] = 1.0 + j * 1e-3;
    f[j] = 0.5f + j * 1e-3f;
  }
  unsigned acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const double x = bump(a[j], i * UNR + u);   // loop-variant: ptxas hoists a pure cvt otherwise
        if (MODE & 1) acc ^= __double2loint(frnd(x));
        if (MODE & 2) acc ^= f2i(x);
        if (MODE & 4) d[j] = fma(d[j], 1.0000001, 1e-9);
        if (MODE & 8) f[j] = ex2(f[j]) * 0.5f;
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
  float fs = 0;
  for (int j = 0; j < CH; ++j) { s += d[j]; fs += f[j]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + (unsigned)s + (unsigned)fs;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int MODE>
void run(const char *name, int sms) {
  const int threads = 256, blocks = sms * 2, iters = 2000;   // all resident at once
  unsigned *out; long long *clk;
  cudaMalloc(&out, sizeof(unsigned) * threads * blocks);
  cudaMalloc(&clk, sizeof(long long));
  k<MODE><<<blocks, threads>>>(10, out, clk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(iters, out, clk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  // warp-level instructions of each tested kind, per SM
  const double warps_per_sm = (double)threads / 32 * 2;
  const double per_kind = warps_per_sm * iters * UNR * CH;
  (void)c;
  // per SM, from the event time at the 1.965 GHz the B200 runs under load (the
  // block-0 clock64 delta undercounts: blocks do not all start together)
  const double cyc = ms * 1e-3 * 1.965e9;
  printf("%-22s %8.3f ms  %6.3f warp-instr/clk/SM per tested kind (%5.1f lanes/clk/SM)\n", name, ms,
         per_kind / cyc, 32.0 * per_kind / cyc);
  cudaFree(out); cudaFree(clk);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  run<4>("DFMA", sms);
  run<1>("FRND.F64", sms);
  run<2>("F2I.F64", sms);
  run<8>("MUFU.EX2", sms);
  run<5>("FRND + DFMA", sms);
  run<6>("F2I + DFMA", sms);
  run<3>("FRND + F2I", sms);
  run<9>("FRND + MUFU", sms);
  run<10>("F2I + MUFU", sms);
  run<7>("FRND + F2I + DFMA", sms);
  return 0;
}
