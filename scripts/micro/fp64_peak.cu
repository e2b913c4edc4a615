// Microbenchmark: FP64 SIMT DFMA vs FP64 tensor-core DMMA (mma.sync m8n8k4) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters) {
  double a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int threads : {256, 512, 1024}) {
      int blocks = sms * (2048 / threads);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * iters * (double)blocks * threads;
      printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(d, iters / 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * (iters / 4) * (double)blocks * (threads / 32);
      printf("DMMA threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    }
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms=%d clock=%d kHz err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
