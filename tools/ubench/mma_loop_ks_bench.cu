// Isolated cost of the packed apply's MMA block body (8 warps, operands resident in shared memory).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__host__ __device__ inline int pk_chunk(int r, int j) { return 8 * (r >> 1) + ((j ^ ((r >> 1) & 3)) + 4 * ((r + j) & 1)); }
__host__ __device__ inline int swz(int r, int c) { return 2 * pk_chunk(r, c >> 1) + (c & 1); }
__device__ __forceinline__ void dmma_pk(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
constexpr int NT8 = 1, MTMAX = 4;
template <int MODE, int KS>
__global__ void __launch_bounds__(256 * KS, 1) k(double* out, int nblk, long long* cyc) {
  extern __shared__ double sm[];
  double* blk = sm;                 // 64 tiles
  double* Dp = sm + 64 * 64;        // 32 k-tiles (ld 256)
  double* Yp = Dp + 256 * 8;
  for (int i = threadIdx.x; i < 64 * 64 + 256 * 9; i += blockDim.x) sm[i] = 1e-3 * (i % 17);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) & 7, hk = threadIdx.x >> 8, qr = lane >> 2, qc = lane & 3;
  constexpr int KK = 8 / KS;
  const int offD = swz(qr, 2 * qc), offT0 = swz(2 * qc, qr), offT1 = swz(2 * qc + 1, qr);
  const int bo = qr * 8 + 2 * qc;
  const int ldD = 256 * 8;
  double acc[NT8][2][MTMAX], accy[MTMAX];
  for (int j = 0; j < MTMAX; ++j) { accy[j] = 0; acc[0][0][j] = 0; acc[0][1][j] = 0; }
  long long t0c = clock64();
  for (int bi = 0; bi < nblk; ++bi) {
    const int gb = (bi % 3) + 1, sb = bi % 2;
    auto step = [&](double (&x0)[2][NT8], double (&x1)[2][NT8], double& xy, double a0, double a1, int kt) {
      const double* db = Dp + kt * 64 + bo;
#pragma unroll
      for (int n = 0; n < NT8; ++n) {
        const double2 bv = *reinterpret_cast<const double2*>(db + n * ldD);
        dmma_pk(x0[0][n], x1[0][n], a0, bv.x);
        dmma_pk(x0[1][n], x1[1][n], a1, bv.y);
      }
      const double2 yv = *reinterpret_cast<const double2*>(Yp + kt * 8 + 2 * qc);
      xy = fma(a1, yv.y, fma(a0, yv.x, xy));
    };
    auto fold = [&](double (&x0)[2][NT8], double (&x1)[2][NT8], double& xy, int jt) {
#pragma unroll
      for (int j = 0; j < MTMAX; ++j)
        if (j == jt) { acc[0][0][j] += x0[0][0] + x0[1][0]; acc[0][1][j] += x1[0][0] + x1[1][0]; accy[j] += xy; }
    };
    double d0[2][NT8] = {}, d1[2][NT8] = {}, dy = 0, t0[2][NT8] = {}, t1[2][NT8] = {}, ty = 0;
    if (MODE == 0) {
#pragma unroll
      for (int k_ = 0; k_ < KK; ++k_) {
        const int kk = hk * KK + k_;
        const double* tpd = blk + (8 * kk + wid) * 64;
        const double2 ad = *reinterpret_cast<const double2*>(tpd + offD);
        step(d0, d1, dy, ad.x, ad.y, 8 * sb + kk);
        const double* tpt = blk + (8 * wid + kk) * 64;
        step(t0, t1, ty, tpt[offT0], tpt[offT1], 8 * gb + kk);
      }
      fold(d0, d1, dy, gb);
      fold(t0, t1, ty, sb);
    } else if (MODE == 1) {
#pragma unroll
      for (int k_ = 0; k_ < KK; ++k_) {
        const int kk = hk * KK + k_;
        const bool dir = kk <= wid;
        const int pos = dir ? 8 * kk - kk * (kk - 1) / 2 + (wid - kk) : 8 * wid - wid * (wid - 1) / 2 + (kk - wid);
        const double* tp = blk + pos * 64;
        step(d0, d1, dy, tp[dir ? offD : offT0], tp[dir ? offD + 1 : offT1], 8 * sb + kk);
      }
      fold(d0, d1, dy, gb);
    } else {
      const double2 ad = *reinterpret_cast<const double2*>(blk + wid * 64 + offD);
      step(d0, d1, dy, ad.x, ad.y, 8 * sb);
      fold(d0, d1, dy, gb);
    }
    __syncwarp();
  }
  long long t1c = clock64();
  double s = 0;
  for (int j = 0; j < MTMAX; ++j) s += acc[0][0][j] + acc[0][1][j] + accy[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0 && hk == 0) cyc[blockIdx.x * 8 + wid] = t1c - t0c;
}
template <int MODE, int KS>
void run(const char* name, double* out, long long* cyc) {
  const int nblk = 1000;
  const size_t smem = (64 * 64 + 256 * 9) * 8;
  cudaFuncSetAttribute(k<MODE, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<MODE, KS><<<148, 256 * KS, smem>>>(out, nblk, cyc);
  cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s: %.0f cycles per block (warp 0), %.0f (warp 7)  [%s]\n", name, (double)h[0] / nblk, (double)h[7] / nblk,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 512 * 8); cudaMalloc(&cyc, 148 * 8 * 8);
  run<0, 1>("off-diagonal block, 8 warps", out, cyc);
  run<0, 2>("off-diagonal block, 16 warps (k split)", out, cyc);
  run<1, 1>("diagonal block, 8 warps", out, cyc);
  run<1, 2>("diagonal block, 16 warps (k split)", out, cyc);
  return 0;
}
