// Microbenchmarks of FP64-pipe throughput for instruction mixes like the
// quadrature loop's.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_chains(int iters, double *out) {
  double a[CH];
  for (int j = 0; j < CH; ++j) a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9;
  const double m = 1.0 + 1e-12, c = 1e-15;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16 / CH; ++u)
#pragma unroll
      for (int j = 0; j < CH; ++j) a[j] = fma(a[j], m, c);
  }
  double s = 0;
  for (int j = 0; j < CH; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 8 chains; each step: DMUL, DADD, DFMA alternate (like the node body)
__global__ void dmix(int iters, double *out) {
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9;
  const double m = 1.0 + 1e-12, c = 1e-15;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = a[j] * m;
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = a[j] + c;
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], m, c);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], m, -c);
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 8 chains of DFMA, each followed by an integer op on the high word (like exp scaling)
__global__ void dfma_int(int iters, double *out) {
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9;
  const double m = 1.0 + 1e-12, c = 1e-15;
  int acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a[j] = fma(a[j], m, c);
        acc += (__double2loint(a[j]) << 3) & 0x7f8;
      }
  }
  double s = acc;
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
float run(K k, int blocks, int threads, int iters, double *out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<blocks, threads>>>(iters / 10, out);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double *out;
  cudaMalloc(&out, 148 * 16 * 1024 * sizeof(double));
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  for (int wps : {4, 8, 16, 32, 48}) {   // warps per SM
    int threads = 128, blocks = 148 * wps / 4;
    double n = (double)blocks * threads * iters * 16;
    float t1 = run(dfma_chains<1>, blocks, threads, iters, out);
    float t2 = run(dfma_chains<2>, blocks, threads, iters, out);
    float t4 = run(dfma_chains<4>, blocks, threads, iters, out);
    float t8 = run(dfma_chains<8>, blocks, threads, iters, out);
    float tm = run(dmix, blocks, threads, iters / 2, out);   // 32 ops per iter
    float ti = run(dfma_int, blocks, threads, iters, out);
    printf("warps/SM=%2d  DFMA Gop/s: 1ch %.0f 2ch %.0f 4ch %.0f 8ch %.0f | mix(DMUL/DADD/DFMA) %.0f | dfma+2int %.0f\n",
           wps, n / t1 / 1e6, n / t2 / 1e6, n / t4 / 1e6, n / t8 / 1e6, n / tm / 1e6, n / ti / 1e6);
  }
  printf("peak at 1.965 GHz: %.0f Gop/s\n", 148 * 64 * 1.965);
  return 0;
}
