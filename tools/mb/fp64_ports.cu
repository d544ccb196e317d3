// FP64-pipe operand microbenchmarks: does the number of distinct register
// operands of a DFMA (register-file read bandwidth) limit its issue rate?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_ports fp64_ports.cu
// Every kernel runs 8 independent chains per thread, 16 FP64 ops per chain per
// iteration; reported in G warp-level FP64 ops/s and % of 148*64*clk.
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8

// 1 fresh operand: a = a*m + c (m, c uniform constants)
__global__ void k_1op(int iters, double *out) {
  double a[CH];
  for (int j = 0; j < CH; ++j) a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9;
  const double m = 1.0 + 1e-12, c = 1e-15;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < CH; ++j) a[j] = fma(a[j], m, c);
  double s = 0;
  for (int j = 0; j < CH; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3 distinct register operands, b/c loop-invariant per chain (reuse possible)
__global__ void k_3op_inv(int iters, double *out) {
  double a[CH], b[CH], c[CH];
  for (int j = 0; j < CH; ++j) {
    a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9;
    b[j] = 1.0 + (j + threadIdx.x) * 1e-13;
    c[j] = (j + 1) * 1e-16 * threadIdx.x;
  }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < CH; ++j) a[j] = fma(a[j], b[j], c[j]);
  double s = 0;
  for (int j = 0; j < CH; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3 fresh operands: two interleaved families, each op reads values written by
// the previous op of other chains (a = a*b + c with b, c from the neighbours)
__global__ void k_3op_fresh(int iters, double *out) {
  double a[CH];
  for (int j = 0; j < CH; ++j) a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < CH; ++j) a[j] = fma(a[(j + 3) % CH], a[(j + 5) % CH], a[j]) * 0.5;
  double s = 0;
  for (int j = 0; j < CH; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 2 fresh operands + immediate: a = a*b + 0.5 (b from a neighbour)
__global__ void k_2op_imm(int iters, double *out) {
  double a[CH];
  for (int j = 0; j < CH; ++j) a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < CH; ++j) a[j] = fma(a[j], a[(j + 3) % CH], -0.5);
  double s = 0;
  for (int j = 0; j < CH; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DADD with 2 fresh operands
__global__ void k_dadd2(int iters, double *out) {
  double a[CH];
  for (int j = 0; j < CH; ++j) a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < CH; ++j) a[j] = a[j] - a[(j + 3) % CH];
  double s = 0;
  for (int j = 0; j < CH; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 1-operand DFMA with one independent integer op per DFMA (like exp's LOP3)
__global__ void k_1op_int1(int iters, double *out) {
  double a[CH];
  int acc[CH];
  for (int j = 0; j < CH; ++j) { a[j] = 1.0 + j * 1e-3 + threadIdx.x * 1e-9; acc[j] = j; }
  const double m = 1.0 + 1e-12, c = 1e-15;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        a[j] = fma(a[j], m, c);
        acc[j] ^= __double2loint(a[j]);
      }
  double s = 0;
  for (int j = 0; j < CH; ++j) s += a[j] + acc[j];
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
  cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  const int iters = 4000;
  const double peak = 148 * 64 * 1.965e9;
  struct { const char *name; void (*k)(int, double *); int ops; } ks[] = {
      {"1op  a=a*m+c", k_1op, 1},        {"3op  loop-invariant b,c", k_3op_inv, 1},
      {"3op  fresh (+DMUL)", k_3op_fresh, 2}, {"2op+imm", k_2op_imm, 1},
      {"DADD 2 fresh", k_dadd2, 1},      {"1op + 1 int", k_1op_int1, 1}};
  for (int wps : {8, 16, 24, 32}) {
    int threads = 128, blocks = 148 * wps / 4;
    for (auto &k : ks) {
      double n = (double)blocks * threads * iters * 16 * CH * k.ops;
      float t = run(k.k, blocks, threads, iters, out);
      printf("warps/SM=%2d %-26s %8.0f Gop/s  %5.1f%% of FP64 pipe\n", wps, k.name, n / t / 1e6,
             100.0 * n / (t * 1e-3) / peak);
    }
  }
  return 0;
}
