// predict_kernels.cu — NEXT-1: the posterior mean and variance of Eq. (4)-(5)
// with the structured covariance K'' of Eq. (28), applied exactly through its
// Woodbury form (reading P22; oracle/predict.py states the algebra):
//   c = R^{-T} y,  zeta_i = u_i^T c_i / sqrt(d_i),  C = I + D^{1/2} M D^{1/2} = L_C L_C^T,
//   per test chunk:  K*_i = k(X_i, X*) on the fly;  W_i = Linv_i K*_i  (FP64 DMMA, lower x dense);
//                    wc_ij = W_ij . c_i,  ww_ij = ||W_ij||^2,  p_ij = u_i . W_ij / sqrt(d_i);
//                    lp = Linv_C p  (DMMA);
//   mean_j = sum_i wc_ij - (sum_i p_ij zeta_i - sum_i lp_ij lz_i),   lz = Linv_C zeta
//   var_j  = alpha - (sum_i ww_ij - (sum_i p_ij^2 - sum_i lp_ij^2))  (+ sigma^2 on request).
// Sums over clusters run in fixed cluster order (deterministic).
#include <cstdint>

#include "common.cuh"
#include "kernels_decl.h"

namespace nugpr {

// K*_i = k(X_i, X*_j) (+ padding rows 0), stored per cluster as ld_i x nt column-major at
// poff_i * nt.  grid = (ceil(nt/32) * ceil(ld_max/32), n_c), 256 threads (32 x 32 tile).
__global__ void __launch_bounds__(256) pred_ks_kernel(const double* X, const double* Xt, int d, LayoutDev L,
                                                      int nt, int ld_max, int kind, double lam, double alpha,
                                                      double* Ks) {
  const int i = blockIdx.y;
  const int ld = L.ld[i];
  const int ntr = (ld_max + 31) / 32;
  const int tr = blockIdx.x % ntr, tc = blockIdx.x / ntr;
  if (tr * 32 >= ld || tc * 32 >= nt) return;
  const int64_t o = L.off[i];
  const int b = static_cast<int>(L.off[i + 1] - o);
  const int r = tr * 32 + (threadIdx.x & 31);
  double* K = Ks + L.poff[i] * nt;
  for (int cc = threadIdx.x >> 5; cc < 32; cc += 8) {
    const int j = tc * 32 + cc;
    if (j >= nt || r >= ld) continue;
    double v = 0.0;
    if (r < b) {
      double sq = 0.0;
      for (int dd = 0; dd < d; ++dd) {
        const double df = __dsub_rn(X[(o + r) * d + dd], Xt[static_cast<int64_t>(j) * d + dd]);
        sq = __dadd_rn(sq, __dmul_rn(df, df));
      }
      v = kval(kind, sq, lam, alpha);
    }
    K[static_cast<int64_t>(j) * ld + r] = v;
  }
}

__device__ __forceinline__ void dmma_p(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Batched lower-triangular x dense: C_g (ld_g x nt) = L_g (ld_g x ld_g, lower, col-major at
// loff_g) * B_g (ld_g x nt col-major at goff_g).  64x64 tiles, 8 warps (2 x 4, warp 32 x 16),
// K staged 16 deep (k <= row-tile end).  grid = (ceil(ld_max/64) * ceil(nt/64), groups).
struct TrmmArgs {
  const double* Lm;
  const double* Bm;
  double* Cm;
  const int32_t* ld;       // per group
  const int64_t* loff;     // per group (element offset of L_g)
  const int64_t* goff;     // per group (element offset of B_g / C_g, in units of rows: offset = goff*nt)
  int nt;
  int ld_max;
};

constexpr int PLD = 68;

__global__ void __launch_bounds__(256) pred_trmm_kernel(TrmmArgs g) {
  const int grp = blockIdx.y;
  const int ld = g.ld[grp];
  const int nrt = (g.ld_max + 63) / 64;
  const int tr = blockIdx.x % nrt, tc = blockIdx.x / nrt;
  const int r0 = tr * 64, c0 = tc * 64;
  if (r0 >= ld || c0 >= g.nt) return;
  const double* Lg = g.Lm + g.loff[grp];
  const double* Bg = g.Bm + g.goff[grp] * g.nt;
  double* Cg = g.Cm + g.goff[grp] * g.nt;
  const int kend = min(ld, r0 + 64);
  __shared__ __align__(16) double As[16 * PLD];
  __shared__ __align__(16) double Bs[16 * PLD];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid & 1, wn = wid >> 1;
  const int qr = lane >> 2, qc = lane & 3;
  double acc[4][2][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) { acc[m][n][0] = 0.0; acc[m][n][1] = 0.0; }
  for (int k0 = 0; k0 < kend; k0 += 16) {
    __syncthreads();
    for (int idx = tid; idx < 16 * 64; idx += 256) {
      const int kk = idx >> 6, x = idx & 63;
      const int k = k0 + kk;
      const int r = r0 + x, c = c0 + x;
      As[kk * PLD + x] = (k < kend && r < ld && k <= r) ? Lg[static_cast<int64_t>(k) * ld + r] : 0.0;
      Bs[kk * PLD + x] = (k < kend && c < g.nt) ? Bg[static_cast<int64_t>(c) * ld + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < 16; k4 += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = As[(k4 + qc) * PLD + wm * 32 + m * 8 + qr];
#pragma unroll
      for (int n = 0; n < 2; ++n) bf[n] = Bs[(k4 + qc) * PLD + wn * 16 + n * 8 + qr];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 2; ++n) dmma_p(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
  }
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = r0 + wm * 32 + m * 8 + qr;
        const int c = c0 + wn * 16 + n * 8 + 2 * qc + e;
        if (r < ld && c < g.nt) Cg[static_cast<int64_t>(c) * ld + r] = acc[m][n][e];
      }
}

// per (cluster i, test column j): wc_ij = W_ij . c_i, ww_ij = ||W_ij||^2, p_ij = u_i . W_ij / sqrt(d_i)
// (one warp per (i, j); outputs [n_c][nt]).  Also zeta_i / d_i on the first column's warps.
__global__ void __launch_bounds__(256) pred_reduce_kernel(LayoutDev L, const double* W, const double* c,
                                                          const double* u, int nt, double* wc, double* ww,
                                                          double* p) {
  const int i = blockIdx.y;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= nt) return;
  const int ld = L.ld[i];
  const int64_t p0 = L.poff[i];
  const double* Wc = W + p0 * nt + static_cast<int64_t>(j) * ld;
  double s1 = 0.0, s2 = 0.0, s3 = 0.0, dd = 0.0;
  for (int r = lane; r < ld; r += 32) {
    const double w = Wc[r];
    const double uu = u[p0 + r];
    s1 = fma(w, c[p0 + r], s1);
    s2 = fma(w, w, s2);
    s3 = fma(uu, w, s3);
    dd = fma(uu, uu, dd);
  }
  s1 = warp_sum(s1); s2 = warp_sum(s2); s3 = warp_sum(s3); dd = warp_sum(dd);
  if (lane == 0) {
    const int64_t o = static_cast<int64_t>(i) * nt + j;
    wc[o] = s1;
    ww[o] = s2;
    p[o] = s3 / sqrt(dd);
  }
}

// zeta_i = u_i . c_i / sqrt(d_i) and sqrt(d_i) (one warp per cluster)
__global__ void pred_zeta_kernel(LayoutDev L, const double* c, const double* u, double* zeta, double* sd) {
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= L.n_c) return;
  const int ld = L.ld[i];
  const int64_t p0 = L.poff[i];
  double s = 0.0, dd = 0.0;
  for (int r = lane; r < ld; r += 32) {
    s = fma(u[p0 + r], c[p0 + r], s);
    dd = fma(u[p0 + r], u[p0 + r], dd);
  }
  s = warp_sum(s); dd = warp_sum(dd);
  if (lane == 0) { sd[i] = sqrt(dd); zeta[i] = s / sqrt(dd); }
}

// C = I + D^{1/2} M D^{1/2} as one ldc x ldc column-major block (identity padding)
__global__ void pred_cmat_kernel(const double* M, const double* sd, int n_c, int ldc, double* Cm) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<int64_t>(ldc) * ldc) return;
  const int r = static_cast<int>(idx % ldc), cc = static_cast<int>(idx / ldc);
  double v = (r == cc) ? 1.0 : 0.0;
  if (r < n_c && cc < n_c) v += sd[r] * M[static_cast<int64_t>(r) * n_c + cc] * sd[cc];
  Cm[idx] = v;
}

// lz = Linv_C zeta (one thread per row; n_c small)
__global__ void pred_lz_kernel(const double* Lc, int ldc, int n_c, const double* zeta, double* lz) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_c) return;
  double s = 0.0;
  for (int k = 0; k <= r; ++k) s = fma(Lc[static_cast<int64_t>(k) * ldc + r], zeta[k], s);
  lz[r] = s;
}

// final: mean/var per test point; p and lp stored [n_c][nt] (p padded to ldc rows for the trmm)
__global__ void pred_final_kernel(int n_c, int nt, int ldc, const double* wc, const double* ww, const double* p,
                                  const double* lp, const double* zeta, const double* lz, double alpha,
                                  double noise_add, double* mean, double* var, int64_t mean_off,
                                  int64_t var_off) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nt) return;
  double swc = 0.0, sww = 0.0, spz = 0.0, slz = 0.0, spp = 0.0, sll = 0.0;
  for (int i = 0; i < n_c; ++i) {
    const double pv = p[static_cast<int64_t>(j) * ldc + i];
    const double lv = lp[static_cast<int64_t>(j) * ldc + i];
    swc += wc[static_cast<int64_t>(i) * nt + j];
    sww += ww[static_cast<int64_t>(i) * nt + j];
    spz = fma(pv, zeta[i], spz);
    slz = fma(lv, lz[i], slz);
    spp = fma(pv, pv, spp);
    sll = fma(lv, lv, sll);
  }
  mean[mean_off + j] = swc - (spz - slz);
  if (var) var[var_off + j] = alpha - (sww - (spp - sll)) + noise_add;
}

// p [n_c][nt] -> column-major ldc x nt (zero padding rows) for the Linv_C trmm
__global__ void pred_pcol_kernel(const double* p, int n_c, int nt, int ldc, double* pc) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<int64_t>(ldc) * nt) return;
  const int r = static_cast<int>(idx % ldc), j = static_cast<int>(idx / ldc);
  pc[idx] = (r < n_c) ? p[static_cast<int64_t>(r) * nt + j] : 0.0;
}

// NEXT-2 (exact structured evaluator): per-cluster c_i . c_i (one warp per cluster)
__global__ void exact_cc_kernel(LayoutDev L, const double* c, double* ccblk) {
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= L.n_c) return;
  const int ld = L.ld[i];
  const int64_t p0 = L.poff[i];
  double s = 0.0;
  for (int r = lane; r < ld; r += 32) s = fma(c[p0 + r], c[p0 + r], s);
  s = warp_sum(s);
  if (lane == 0) ccblk[i] = s;
}

// quad = c^T c - (zeta^T zeta - ||Linv_C zeta||^2), logdet = logdet_R + log|C|, L = (quad + logdet + n log 2 pi)/2
// (one CTA; fixed-order strided partials then a fixed tree -> deterministic)
__global__ void __launch_bounds__(256) exact_final_kernel(int n_c, int64_t n, const double* ccblk, const double* zeta,
                                                          const double* lz, const double* logdet_R,
                                                          const double* logdet_C, double* out) {
  __shared__ double red[3][256];
  double a = 0.0, b = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < n_c; i += 256) {
    a += ccblk[i];
    b = fma(zeta[i], zeta[i], b);
    c = fma(lz[i], lz[i], c);
  }
  red[0][threadIdx.x] = a; red[1][threadIdx.x] = b; red[2][threadIdx.x] = c;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int q = 0; q < 3; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double quad = red[0][0] - (red[1][0] - red[2][0]);
    const double logdet = logdet_R[0] + logdet_C[0];
    out[0] = 0.5 * (quad + logdet + static_cast<double>(n) * 1.8378770664093454836);   // log(2 pi)
    out[1] = quad;
    out[2] = logdet;
    out[3] = logdet_C[0];
  }
}

void launch_exact_final(const LayoutDev& L, const double* c, const double* zeta, const double* lz,
                        const double* logdet_R, const double* logdet_C, double* ccblk, int64_t n, double* out,
                        cudaStream_t s) {
  exact_cc_kernel<<<(L.n_c + 7) / 8, 256, 0, s>>>(L, c, ccblk);
  exact_final_kernel<<<1, 256, 0, s>>>(L.n_c, n, ccblk, zeta, lz, logdet_R, logdet_C, out);
  note_launch(2); post_launch("exact_final");
}

// ------------------------------------------------------------------------------- launchers
void launch_pred_ks(const double* X, const double* Xt, int d, const LayoutDev& L, int nt, int ld_max, int kind,
                    double lam, double alpha, double* Ks, cudaStream_t s) {
  const int grid_x = ((ld_max + 31) / 32) * ((nt + 31) / 32);
  pred_ks_kernel<<<dim3(grid_x, L.n_c), 256, 0, s>>>(X, Xt, d, L, nt, ld_max, kind, lam, alpha, Ks);
  note_launch(); post_launch("pred_ks_kernel");
}

void launch_pred_trmm(const double* Lm, const double* Bm, double* Cm, const int32_t* ld, const int64_t* loff,
                      const int64_t* goff, int groups, int nt, int ld_max, cudaStream_t s) {
  TrmmArgs g{Lm, Bm, Cm, ld, loff, goff, nt, ld_max};
  const int grid_x = ((ld_max + 63) / 64) * ((nt + 63) / 64);
  pred_trmm_kernel<<<dim3(grid_x, groups), 256, 0, s>>>(g);
  note_launch(); post_launch("pred_trmm_kernel");
}

void launch_pred_reduce(const LayoutDev& L, const double* W, const double* c, const double* u, int nt, double* wc,
                        double* ww, double* p, cudaStream_t s) {
  pred_reduce_kernel<<<dim3((nt + 7) / 8, L.n_c), 256, 0, s>>>(L, W, c, u, nt, wc, ww, p);
  note_launch(); post_launch("pred_reduce_kernel");
}

void launch_pred_setup(const LayoutDev& L, const double* c, const double* u, const double* M, int ldc, double* zeta,
                       double* sd, double* Cm, cudaStream_t s) {
  pred_zeta_kernel<<<(L.n_c + 7) / 8, 256, 0, s>>>(L, c, u, zeta, sd);
  const int64_t tot = static_cast<int64_t>(ldc) * ldc;
  pred_cmat_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(M, sd, L.n_c, ldc, Cm);
  note_launch(2); post_launch("pred_setup");
}

void launch_pred_lz(const double* Lc, int ldc, int n_c, const double* zeta, double* lz, cudaStream_t s) {
  pred_lz_kernel<<<(n_c + 127) / 128, 128, 0, s>>>(Lc, ldc, n_c, zeta, lz);
  note_launch(); post_launch("pred_lz_kernel");
}

void launch_pred_pcol(const double* p, int n_c, int nt, int ldc, double* pc, cudaStream_t s) {
  const int64_t tot = static_cast<int64_t>(ldc) * nt;
  pred_pcol_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(p, n_c, nt, ldc, pc);
  note_launch(); post_launch("pred_pcol_kernel");
}

void launch_pred_final(int n_c, int nt, int ldc, const double* wc, const double* ww, const double* p, const double* lp,
                       const double* zeta, const double* lz, double alpha, double noise_add, double* mean, double* var,
                       int64_t mean_off, int64_t var_off, cudaStream_t s) {
  pred_final_kernel<<<(nt + 127) / 128, 128, 0, s>>>(n_c, nt, ldc, wc, ww, p, lp, zeta, lz, alpha, noise_add, mean, var,
                                                   mean_off, var_off);
  note_launch(); post_launch("pred_final_kernel");
}

}  // namespace nugpr
