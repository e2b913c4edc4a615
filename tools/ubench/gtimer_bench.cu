#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, unsigned long long* g) {
  long long c0 = clock64();
  unsigned long long s = 0;
  for (int i = 0; i < 1000; ++i) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    s += t;
    if ((threadIdx.x & 31) == 0) g[i] = t;
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = s; }
}
int main() {
  long long* o; unsigned long long* g; cudaMalloc(&o, 16); cudaMalloc(&g, 8000 * 8);
  k<<<1, 32>>>(o, g); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, g); cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  unsigned long long hg[1000]; cudaMemcpy(hg, g, 8000, cudaMemcpyDeviceToHost);
  printf("globaltimer read+store: %.1f cycles each; timer span %llu ns over 1000 reads\n", h[0] / 1000.0, hg[999] - hg[0]);
}
