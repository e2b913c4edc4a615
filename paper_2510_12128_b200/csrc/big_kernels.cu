// big_kernels.cu — rows A1 and A3 for clusters larger than the single-CTA kernels handle
// (ld_max > 512: config C4's uneven k-means clusters, up to ~4.3k points; the paper's own
// datasets use b ~ 1600).
//
// A1, blocked over 64-wide panels, batched over all clusters, K_i assembled in place:
//   for k0 = 0, 64, ...:  diag  : L_kk = chol(A_kk) in shared memory, Xd_k = L_kk^{-1} kept,
//                                 logdet partial 2 sum log diag(L_kk), status on a bad pivot
//                         trsm  : L_21 = A_21 Xd_k^T                         (64-row tiles)
//                         syrk  : A_22 -= L_21 L_21^T (lower 64x64 tiles, FP64 DMMA)
//   zero the strict upper triangle, then Linv = L^{-1} in place by 64-row panels I:
//                         invy  : Y = L[I, 0:I0] X[0:I0, 0:I0]    (DMMA, X already inverted)
//                         invx  : X[I, 0:I0] = -Xd_I Y            (DMMA)
//                         invd  : X_II = Xd_I
//   and u = Linv 1_b.
// A3: a row-tiled apply (64 rows x c columns per CTA) that streams the 64 contiguous columns of
// the symmetric block B_i (= its rows) against D_i in 64-deep k chunks, with the same combine /
// epilogue contract as the other apply kernels and per-tile partial sums.
#include <cstdint>

#include "cg_fin.cuh"
#include "common.cuh"
#include "kernels_decl.h"

namespace nugpr {

constexpr int BNB = 64;                   // panel / tile size
constexpr int BLDS = BNB + 4;             // padded smem stride (4 mod 16 in doubles -> conflict-free fragments)

struct BigArgs {
  double* A;                 // block storage (K in, Linv out)
  const int64_t* off;
  const int64_t* poff;
  const int64_t* boff;
  const int32_t* ld;
  const int32_t* list;       // NULL => blockIdx.y is the cluster
  int32_t* status;
  double* logdet_blk;
  double* u;
  double* Xs;                // per cluster: ld_max/64 diag-block inverses (64x64, col-major)
  double* Ys;                // per cluster: 64 x ld_max scratch (inverse step)
  int ld_max;
  int k0;                    // panel start (Cholesky step / inverse row panel I0)
};

__device__ __forceinline__ int big_cluster(const BigArgs& g) { return g.list ? g.list[blockIdx.y] : blockIdx.y; }

__device__ __forceinline__ void dmma_b(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------------- diag
__global__ void __launch_bounds__(256) big_diag_kernel(BigArgs g) {
  const int i = big_cluster(g);
  const int ld = g.ld[i];
  const int k0 = g.k0;
  if (k0 >= ld) return;
  const int nb = min(BNB, ld - k0);
  const int b = static_cast<int>(g.off[i + 1] - g.off[i]);
  double* A = g.A + g.boff[i];
  extern __shared__ double bsm[];
  double* Ls = bsm;                         // column-major, stride 65
  double* Xd = bsm + BNB * (BNB + 1);
  __shared__ int fail;
  __shared__ double red[8];
  const int tid = threadIdx.x;
  if (tid == 0) fail = 0;
  for (int idx = tid; idx < nb * nb; idx += 256) {
    const int c = idx / nb, r = idx % nb;
    Ls[c * (BNB + 1) + r] = (r >= c) ? A[static_cast<int64_t>(k0 + c) * ld + k0 + r] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (tid == 0) {
      double piv = Ls[j * (BNB + 1) + j];
      if (!(piv > 0.0)) { fail = 1; piv = 1.0; }
      Ls[j * (BNB + 1) + j] = sqrt(piv);
    }
    __syncthreads();
    const double inv = 1.0 / Ls[j * (BNB + 1) + j];
    for (int r = j + 1 + tid; r < nb; r += 256) Ls[j * (BNB + 1) + r] *= inv;
    __syncthreads();
    const int m = nb - j - 1;
    for (int idx = tid; idx < m * m; idx += 256) {
      const int c = j + 1 + idx / m, r = j + 1 + idx % m;
      if (r >= c) Ls[c * (BNB + 1) + r] -= Ls[j * (BNB + 1) + r] * Ls[j * (BNB + 1) + c];
    }
    __syncthreads();
  }
  // logdet partial over the real rows of this panel
  double ls = 0.0;
  for (int r = tid; r < nb; r += 256)
    if (k0 + r < b) ls += log(Ls[r * (BNB + 1) + r]);
  ls = warp_sum(ls);
  if ((tid & 31) == 0) red[tid >> 5] = ls;
  // inverse of the diagonal block: thread j solves L x = e_j
  if (tid < nb) {
    const int j = tid;
    for (int r = 0; r < nb; ++r) {
      double v = 0.0;
      if (r >= j) {
        v = (r == j) ? 1.0 : 0.0;
        for (int k = j; k < r; ++k) v -= Ls[k * (BNB + 1) + r] * Xd[j * (BNB + 1) + k];
        v /= Ls[r * (BNB + 1) + r];
      }
      Xd[j * (BNB + 1) + r] = v;
    }
  }
  __syncthreads();
  if (tid == 0) {
    double s_ = 0.0;
    for (int w = 0; w < 8; ++w) s_ += red[w];
    if (k0 == 0) { g.logdet_blk[i] = 2.0 * s_; g.status[i] = fail; }
    else { g.logdet_blk[i] += 2.0 * s_; g.status[i] |= fail; }
  }
  for (int idx = tid; idx < nb * nb; idx += 256) {
    const int c = idx / nb, r = idx % nb;
    if (r >= c) A[static_cast<int64_t>(k0 + c) * ld + k0 + r] = Ls[c * (BNB + 1) + r];
  }
  double* X = g.Xs + static_cast<int64_t>(i) * g.ld_max * BNB + static_cast<int64_t>(k0 / BNB) * BNB * BNB;
  for (int idx = tid; idx < BNB * BNB; idx += 256) {
    const int c = idx / BNB, r = idx % BNB;
    X[c * BNB + r] = (r < nb && c < nb) ? Xd[c * (BNB + 1) + r] : 0.0;
  }
}

// ---------------------------------------------------------------------------------- trsm
// L21[rows, k0:k0+nb] = A21 Xd^T, 64-row tile per CTA (SIMT, 4x4 register tiles), in place.
__global__ void __launch_bounds__(256) big_trsm_kernel(BigArgs g) {
  const int i = big_cluster(g);
  const int ld = g.ld[i];
  const int k0 = g.k0;
  const int r0 = k0 + BNB + blockIdx.x * BNB;
  if (k0 + BNB >= ld || r0 >= ld) return;
  const int nb = min(BNB, ld - k0);          // == BNB here
  const int nr = min(BNB, ld - r0);
  double* A = g.A + g.boff[i];
  const double* X = g.Xs + static_cast<int64_t>(i) * g.ld_max * BNB + static_cast<int64_t>(k0 / BNB) * BNB * BNB;
  extern __shared__ double bsm[];
  double* Ps = bsm;                         // P[r][k] at k*BLDS + r
  double* Xt = bsm + BNB * BLDS;            // Xd[c][k] at k*BLDS + c
  const int tid = threadIdx.x;
  for (int idx = tid; idx < BNB * BNB; idx += 256) {
    const int k = idx / BNB, r = idx % BNB;
    Ps[k * BLDS + r] = (r < nr && k < nb) ? A[static_cast<int64_t>(k0 + k) * ld + r0 + r] : 0.0;
    Xt[k * BLDS + r] = X[k * BNB + r];      // column k of Xd: Xd[r][k], i.e. Xt[k][c=r]
  }
  __syncthreads();
  const int tx = tid & 15, ty = tid >> 4;   // rows tx*4.., cols ty*4..
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
  for (int k = 0; k < BNB; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) av[x] = Ps[k * BLDS + tx * 4 + x];
#pragma unroll
    for (int y = 0; y < 4; ++y) bv[y] = Xt[k * BLDS + ty * 4 + y];   // Xd[c][k]
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
  }
  __syncthreads();
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    const int c = ty * 4 + y;
    if (c >= nb) continue;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int r = tx * 4 + x;
      if (r < nr) A[static_cast<int64_t>(k0 + c) * ld + r0 + r] = acc[x][y];
    }
  }
}

// ------------------------------------------------------------------- DMMA 64x64 tile GEMMs
// One 64x64 output tile per CTA, 8 warps as 2 x 4, warp tile 32 x 16, K staged 16 deep.
// opA(r, k) and opB(k, c) are read through the mode's addressing; out += sgn * opA opB.
enum BigMode { BM_SYRK = 0, BM_INVY = 1, BM_INVX = 2 };

template <int MODE>
__global__ void __launch_bounds__(256) big_gemm_kernel(BigArgs g) {
  const int i = big_cluster(g);
  const int ld = g.ld[i];
  const int k0 = g.k0;
  double* A = g.A + g.boff[i];
  int R, Cc, kbeg, kend;
  if (MODE == BM_SYRK) {
    const int t0 = k0 + BNB;
    if (t0 >= ld) return;
    const int nt = (ld - t0 + BNB - 1) / BNB;
    const int t = blockIdx.x;
    if (t >= nt * (nt + 1) / 2) return;
    int bi = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const int bj = t - bi * (bi + 1) / 2;
    R = t0 + bi * BNB; Cc = t0 + bj * BNB; kbeg = 0; kend = BNB;
  } else {
    const int I0 = k0;
    if (I0 >= ld) return;
    const int c0 = blockIdx.x * BNB;
    if (c0 >= I0) return;
    R = I0; Cc = c0;
    if (MODE == BM_INVY) { kbeg = c0; kend = I0; } else { kbeg = 0; kend = BNB; }
  }
  const double* Xd = g.Xs + static_cast<int64_t>(i) * g.ld_max * BNB + static_cast<int64_t>(k0 / BNB) * BNB * BNB;
  double* Y = g.Ys + static_cast<int64_t>(i) * g.ld_max * BNB;   // Y[c][r] at c*64 + r
  // element loaders
  auto opA = [&](int r, int k) -> double {      // r in [0,64), absolute k
    const int rr = R + r;
    if (rr >= ld) return 0.0;
    if (MODE == BM_SYRK) return A[static_cast<int64_t>(k0 + k) * ld + rr];         // P[rr][k]
    if (MODE == BM_INVY) return A[static_cast<int64_t>(k) * ld + rr];              // L[I0+r][k]
    return (k <= r) ? Xd[k * BNB + r] : 0.0;                                      // Xd[r][k]
  };
  auto opB = [&](int k, int c) -> double {      // c in [0,64)
    const int cc = Cc + c;
    if (MODE == BM_SYRK) return (cc < ld) ? A[static_cast<int64_t>(k0 + k) * ld + cc] : 0.0;   // P[cc][k]
    if (MODE == BM_INVY) return (cc < g.k0 && k >= cc) ? A[static_cast<int64_t>(cc) * ld + k] : 0.0;  // X[k][cc]
    return (cc < g.k0) ? Y[static_cast<int64_t>(cc) * BNB + k] : 0.0;                           // Y[k][cc]
  };
  __shared__ __align__(16) double As[16 * BLDS];
  __shared__ __align__(16) double Bs[16 * BLDS];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid & 1, wn = wid >> 1;
  const int qr = lane >> 2, qc = lane & 3;
  double acc[4][2][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) { acc[m][n][0] = 0.0; acc[m][n][1] = 0.0; }
  for (int kk = kbeg; kk < kend; kk += 16) {
    __syncthreads();
    for (int idx = tid; idx < 16 * BNB; idx += 256) {
      const int k = idx / BNB, x = idx % BNB;
      const bool kin = kk + k < kend;
      As[k * BLDS + x] = kin ? opA(x, kk + k) : 0.0;
      Bs[k * BLDS + x] = kin ? opB(kk + k, x) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < 16; k4 += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = As[(k4 + qc) * BLDS + wm * 32 + m * 8 + qr];
#pragma unroll
      for (int n = 0; n < 2; ++n) bf[n] = Bs[(k4 + qc) * BLDS + wn * 16 + n * 8 + qr];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 2; ++n) dmma_b(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
  }
  // write-back
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = wm * 32 + m * 8 + qr;
        const int c = wn * 16 + n * 8 + 2 * qc + e;
        const int rr = R + r, cc = Cc + c;
        const double v = acc[m][n][e];
        if (MODE == BM_SYRK) {
          if (rr < ld && cc < ld && rr >= cc) A[static_cast<int64_t>(cc) * ld + rr] -= v;
        } else if (MODE == BM_INVY) {
          if (cc < g.k0) Y[static_cast<int64_t>(cc) * BNB + r] = v;
        } else {
          if (rr < ld && cc < g.k0) A[static_cast<int64_t>(cc) * ld + rr] = -v;
        }
      }
}

// X_II = Xd_I (lower; the strict upper part of the block is already zero)
__global__ void __launch_bounds__(256) big_invd_kernel(BigArgs g) {
  const int i = big_cluster(g);
  const int ld = g.ld[i];
  const int I0 = g.k0;
  if (I0 >= ld) return;
  const int nb = min(BNB, ld - I0);
  double* A = g.A + g.boff[i];
  const double* Xd = g.Xs + static_cast<int64_t>(i) * g.ld_max * BNB + static_cast<int64_t>(I0 / BNB) * BNB * BNB;
  for (int idx = threadIdx.x; idx < nb * nb; idx += 256) {
    const int c = idx / nb, r = idx % nb;
    if (r >= c) A[static_cast<int64_t>(I0 + c) * ld + I0 + r] = Xd[c * BNB + r];
  }
}

// strict upper triangle := 0 (64x64 tiles, grid.x = tile index)
__global__ void __launch_bounds__(256) big_zero_upper_kernel(BigArgs g) {
  const int i = big_cluster(g);
  const int ld = g.ld[i];
  const int nt = (ld + BNB - 1) / BNB;
  const int t = blockIdx.x;
  if (t >= nt * nt) return;
  const int tr = t % nt, tc = t / nt;
  if (tc < tr) return;
  double* A = g.A + g.boff[i];
  for (int idx = threadIdx.x; idx < BNB * BNB; idx += 256) {
    const int c = tc * BNB + idx / BNB, r = tr * BNB + idx % BNB;
    if (r < ld && c < ld && c > r) A[static_cast<int64_t>(c) * ld + r] = 0.0;
  }
}

// u = Linv 1_b (row sums over the real columns), padding rows 0
__global__ void __launch_bounds__(256) big_u_kernel(BigArgs g) {
  const int i = big_cluster(g);
  const int ld = g.ld[i];
  const int b = static_cast<int>(g.off[i + 1] - g.off[i]);
  const int r = blockIdx.x * 256 + threadIdx.x;
  if (r >= ld) return;
  const double* A = g.A + g.boff[i];
  double acc = 0.0;
  if (r < b)
    for (int k = 0; k <= r; ++k) acc += A[static_cast<int64_t>(k) * ld + r];
  g.u[g.poff[i] + r] = acc;
}

size_t big_scratch_doubles(int n_c, int ld_max) {
  const size_t per = static_cast<size_t>(((ld_max + BNB - 1) / BNB) * BNB) * BNB;
  return 2 * per * n_c;   // Xs + Ys
}

// Full big-block build of the clusters in `list` (NULL: all): Cholesky, logdet partials, status,
// then (for the clusters that did not fail) Linv in place and u.  The host launches the panel
// steps; everything is enqueued on s.
void launch_big_chol_trtri(double* A, const LayoutDev& L, const int32_t* list, int nlist, int ld_max,
                           int32_t* status, double* logdet_blk, double* u, double* scratch, cudaStream_t s) {
  const int ny = list ? nlist : L.n_c;
  const int ldr = ((ld_max + BNB - 1) / BNB) * BNB;
  BigArgs g;
  g.A = A; g.off = L.off; g.poff = L.poff; g.boff = L.boff; g.ld = L.ld; g.list = list; g.status = status;
  g.logdet_blk = logdet_blk; g.u = u; g.ld_max = ldr;
  g.Xs = scratch;
  g.Ys = scratch + static_cast<size_t>(ldr) * BNB * L.n_c;
  const int ntl = ldr / BNB;
  const size_t sm_diag = sizeof(double) * 2 * BNB * (BNB + 1), sm_trsm = sizeof(double) * 2 * BNB * BLDS;
  smem_optin(reinterpret_cast<const void*>(big_diag_kernel));
  smem_optin(reinterpret_cast<const void*>(big_trsm_kernel));
  for (int k0 = 0; k0 < ld_max; k0 += BNB) {
    g.k0 = k0;
    big_diag_kernel<<<dim3(1, ny), 256, sm_diag, s>>>(g);
    const int rows_below = ldr - k0 - BNB;
    if (rows_below > 0) {
      big_trsm_kernel<<<dim3(rows_below / BNB, ny), 256, sm_trsm, s>>>(g);
      const int nt = rows_below / BNB;
      big_gemm_kernel<BM_SYRK><<<dim3(nt * (nt + 1) / 2, ny), 256, 0, s>>>(g);
      note_launch(2);
    }
    note_launch();
  }
  big_zero_upper_kernel<<<dim3(ntl * ntl, ny), 256, 0, s>>>(g);
  note_launch();
  // (a failed cluster's inverse is garbage but unused: the host re-runs it with jitter)
  for (int I0 = 0; I0 < ld_max; I0 += BNB) {
    g.k0 = I0;
    if (I0 > 0) {
      big_gemm_kernel<BM_INVY><<<dim3(I0 / BNB, ny), 256, 0, s>>>(g);
      big_gemm_kernel<BM_INVX><<<dim3(I0 / BNB, ny), 256, 0, s>>>(g);
      note_launch(2);
    }
    big_invd_kernel<<<dim3(1, ny), 256, 0, s>>>(g);
    note_launch();
  }
  big_u_kernel<<<dim3((ld_max + 255) / 256, ny), 256, 0, s>>>(g);
  note_launch(); post_launch("big_chol_trtri");
}

// ---------------------------------------------------------------------------------- apply
// Row-tiled apply for any ld (big mode: tiles are 64-row pieces of clusters).  CTA = tile t
// (cluster i, rows [r0, r0+nr)): acc[r][c] = sum_k B_i[k][r0+r] D_i[k][c] (B symmetric), k in
// 64-deep chunks staged in shared memory with plain coalesced loads (each chunk: 64 column
// segments of B and the c columns of D).  Epilogue and partial sums as in apply_kernel; the
// S / dot partials are per tile (lowrank sums a cluster's tiles through tile0).
// (not volatile: a pure function of its operands)
__device__ __forceinline__ void dmma_big(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NCP>
__global__ void __launch_bounds__(256) apply_big_kernel(ApplyArgs a) {
  if (a.gate && !a.st->any_active) return;
  const int t = blockIdx.x;
  const TileDesc td = a.L.tiles[t];
  const int i = td.blk;
  const int ld = a.L.ld[i];
  const int r0 = td.row0, nr = td.nrows;
  const int64_t p0 = a.L.poff[i];
  const int64_t n_pad = a.L.n_pad;
  const int ncol = a.ncol;
  const EvalParams* P = a.prm;
  const int par = a.st->par;
  const double* B = P->B;
  const bool useB = (B != nullptr);
  const double* Bi = useB ? B + a.L.boff[i] : nullptr;
  const double* Pold = a.fuse_p ? a.Pbuf[par] : nullptr;
  double* Pnew = a.fuse_p ? a.Pbuf[par ^ 1] : nullptr;
  const double* P2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.P2;
  const double* Y2 = a.use_par_p2 ? a.Pbuf[par ^ 1] : a.Y2;
  __shared__ double Bs[BNB * BLDS];          // Bs[k][r] = B_i[k0+k][r0+r]
  __shared__ double Ds[BNB * NCP];           // Ds[k][c] = D_i[k0+k][c]
  __shared__ double cb[2 * MAXC];
  __shared__ double sred[8 * MAXC];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < MAXC) {
    cb[tid] = (tid < ncol) ? a.st->beta[tid] : 0.0;
    cb[MAXC + tid] = (tid < ncol) ? static_cast<double>(a.st->active[tid]) : 0.0;
  }
  __syncthreads();
  // D value with the fused search-direction update
  auto dval = [&](int c, int64_t gi) -> double {
    double v = a.D[gi];
    if (a.fuse_p) {
      const double po = Pold[gi];
      v = (cb[MAXC + c] != 0.0) ? v + cb[c] * po : po;
    }
    return v;
  };
  // thread -> (row r = tid % 64, column group cg = tid / 64): columns cg, cg+4, ...
  const int r = tid & 63, cg = tid >> 6;
  constexpr int CPT = (NCP + 3) / 4;
  double acc[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) acc[q] = 0.0;
  const int qr = lane >> 2, qc = lane & 3;
  double m0[2] = {0.0, 0.0}, m1[2] = {0.0, 0.0}, my = 0.0;   // (NCP == 10) DMMA accumulators
  __shared__ double Accs[(NCP == 10) ? BNB * NCP : 1];
  if (useB) {
    // register double buffering: chunk k0+64 is loaded while chunk k0 is multiplied
    constexpr int NBV = BNB * BNB / 256, NDV = (BNB * NCP + 255) / 256;
    double rbv[NBV], rdv[NDV];
    auto gload = [&](int k0) {
      const int kc = min(BNB, ld - k0);
#pragma unroll
      for (int u = 0; u < NBV; ++u) {
        const int idx = tid + u * 256;
        const int rr = idx / BNB, k = idx % BNB;
        rbv[u] = (rr < nr && k < kc) ? Bi[static_cast<int64_t>(r0 + rr) * ld + k0 + k] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < NDV; ++u) {
        const int idx = tid + u * 256;
        const int c = idx / BNB, k = idx % BNB;
        rdv[u] = (idx < BNB * NCP && c < ncol && k < kc) ? dval(c, c * n_pad + p0 + k0 + k) : 0.0;
      }
    };
    auto sstore = [&]() {
#pragma unroll
      for (int u = 0; u < NBV; ++u) {
        const int idx = tid + u * 256;
        Bs[(idx % BNB) * BLDS + idx / BNB] = rbv[u];
      }
#pragma unroll
      for (int u = 0; u < NDV; ++u) {
        const int idx = tid + u * 256;
        if (idx < BNB * NCP) Ds[(idx % BNB) * NCP + idx / BNB] = rdv[u];
      }
    };
    gload(0);
    for (int k0 = 0; k0 < ld; k0 += BNB) {
      const int kc = min(BNB, ld - k0);
      __syncthreads();
      sstore();
      __syncthreads();
      if (k0 + BNB < ld) gload(k0 + BNB);
      if constexpr (NCP == 10) {
        // y + 8 probe columns: the 8 probes on the FP64 tensor pipe (warp w: rows 8w..8w+7 as one m8
        // tile, the probes as one n8 tile, two independent accumulator chains over k), the y column
        // by DFMA on the same A fragment; each B element is read once per warp from shared memory
#pragma unroll 4
        for (int k4 = 0; k4 < kc; k4 += 8) {
          const int ka = k4 + qc, kb = k4 + 4 + qc;
          const double aa = Bs[ka * BLDS + 8 * wid + qr], ab = Bs[kb * BLDS + 8 * wid + qr];
          const double ba = Ds[ka * NCP + 1 + qr], bb = Ds[kb * NCP + 1 + qr];
          dmma_big(m0[0], m0[1], aa, ba);
          dmma_big(m1[0], m1[1], ab, bb);
          my = fma(ab, Ds[kb * NCP], fma(aa, Ds[ka * NCP], my));
        }
      } else {
        for (int k = 0; k < kc; ++k) {
          const double bv = Bs[k * BLDS + r];
#pragma unroll
          for (int q = 0; q < CPT; ++q) acc[q] = fma(bv, Ds[k * NCP + min(cg + 4 * q, NCP - 1)], acc[q]);
        }
      }
    }
    if constexpr (NCP == 10) {
      // fragments -> (row, column) layout of the epilogue through shared memory
      my += __shfl_xor_sync(0xffffffffu, my, 1);
      my += __shfl_xor_sync(0xffffffffu, my, 2);
      const int row = 8 * wid + qr;
      if (qc == 0) Accs[row * NCP] = my;
      Accs[row * NCP + 1 + 2 * qc] = m0[0] + m1[0];
      Accs[row * NCP + 2 + 2 * qc] = m0[1] + m1[1];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < CPT; ++q) acc[q] = Accs[r * NCP + min(cg + 4 * q, NCP - 1)];
    }
  }
  // epilogue for (row r, columns cg + 4q)
  double ep[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) ep[q] = 0.0;
  if (r < nr) {
    const int rr = r0 + r;
    const double bi = P->b0 + P->b1 * a.jitter[i];
    const double uu = a.u[p0 + rr];
    const double* Tq = a.Tbuf + static_cast<int64_t>(i) * MAXC;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int c = cg + 4 * q;
      if (c >= ncol) continue;
      const int64_t gi = c * n_pad + p0 + rr;
      const double d = dval(c, gi);
      if (a.fuse_p) Pnew[gi] = d;
      double val = P->a * d;
      if (useB) val += bi * acc[q];
      val += uu * (P->mscale * Tq[c]);
      double o = a.cA[c] * val + a.cV[c] * d;
      if (P2) o += a.cP[c] * P2[gi];
      a.out[gi] = o;
      ep[q] = o * ((a.epi == EPI_S) ? uu : Y2[gi]);
    }
  }
  // per-tile column sums: warp sums (the warp's lanes share cg), then fixed-order over warps
#pragma unroll
  for (int q = 0; q < CPT; ++q) ep[q] = warp_sum(ep[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < CPT; ++q) sred[wid * MAXC + q] = ep[q];
  __syncthreads();
  if (tid < ncol) {
    const int c = tid, g4 = c & 3, q = c >> 2;   // column c lives in warps of group g4 (2 warps)
    const double s = sred[(2 * g4) * MAXC + q] + sred[(2 * g4 + 1) * MAXC + q];
    if (a.epi == EPI_S) a.Sout[t * MAXC + c] = s;
    else a.dots[t * MAXC + c] = s;
  }
  // finaliser (last CTA)
  if (a.fin != FIN_NONE) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&a.st->ticket[a.fin], 1u) == gridDim.x - 1);
    __syncthreads();
    if (s_last) {
      __threadfence();
      fin_alpha_trace_body(a.fin, a.st, a.dots, a.L.n_tiles, ncol, a.alpha_hist, a.hist_stride, 8);
      __syncthreads();
      if (tid == 0) a.st->ticket[a.fin] = 0;
    }
  }
}

void launch_apply_big(const ApplyArgs& a, int ncp, cudaStream_t s) {
  switch (ncp) {
    case 2: apply_big_kernel<2><<<a.L.n_tiles, 256, 0, s>>>(a); break;
    case 4: apply_big_kernel<4><<<a.L.n_tiles, 256, 0, s>>>(a); break;
    case 6: apply_big_kernel<6><<<a.L.n_tiles, 256, 0, s>>>(a); break;
    case 8: apply_big_kernel<8><<<a.L.n_tiles, 256, 0, s>>>(a); break;
    case 10: apply_big_kernel<10><<<a.L.n_tiles, 256, 0, s>>>(a); break;
    case 12: apply_big_kernel<12><<<a.L.n_tiles, 256, 0, s>>>(a); break;
    case 14: apply_big_kernel<14><<<a.L.n_tiles, 256, 0, s>>>(a); break;
    default: apply_big_kernel<16><<<a.L.n_tiles, 256, 0, s>>>(a); break;
  }
  note_launch(); post_launch("apply_big_kernel");
}

}  // namespace nugpr
