// DMMA m8n8k4 latency / throughput probe: W warps per CTA, C independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int C>
__global__ void k(double* out, int iters, double a, double b) {
  double d0[C], d1[C];
  for (int c = 0; c < C; ++c) { d0[c] = threadIdx.x; d1[c] = c; }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < C; ++c) dmma(d0[c], d1[c], a, b);
  double s = 0;
  for (int c = 0; c < C; ++c) s += d0[c] + d1[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C>
void run(int warps, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  k<C><<<148, warps * 32>>>(out, 16, 1.0, 1e-9);
  cudaEventRecord(e0);
  k<C><<<148, warps * 32>>>(out, iters, 1.0, 1e-9);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = 148.0 * warps * iters * C;
  double tf = n * 512 / (ms * 1e-3) / 1e12;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc_per_dmma_smsp = (ms * 1e-3) * clk * 1e3 / (n / 148 / 4);
  printf("chains %d warps/CTA %2d: %.2f TF/s  %.1f cycles/DMMA/SMSP  (%.1f cycles latency per chain step)\n", C, warps, tf,
         cyc_per_dmma_smsp, (ms * 1e-3) * clk * 1e3 / iters);
}
int main() {
  double* out; cudaMalloc(&out, 148 * 1024 * 8);
  for (int w : {1, 4, 8, 16, 32}) { run<1>(w, out); run<2>(w, out); run<4>(w, out); run<8>(w, out); }
  return 0;
}
