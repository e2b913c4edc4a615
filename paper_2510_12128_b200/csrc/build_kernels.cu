// build_kernels.cu — rows A1/A2 of SURVEY §8(a): on-the-fly kernel-block assembly,
// batched per-cluster Cholesky + triangular inverse, batched FP64 GEMMs for
// H_i = R_i^{-T} R_i^{-1} and G_i(theta') = R_i^{-T} K_i(theta') R_i^{-1}, K_rep and the
// Lanczos lambda_0 = lambda_min(K_rep).
//
// Notation: L_i = R_i^T is the lower Cholesky factor of K_i, Linv_i = L_i^{-1} = R_i^{-T}.
// Then u_i = Linv_i 1 (Eq. 21), c_i = Linv_i y_i, H_i = Linv_i Linv_i^T,
// G_i = Linv_i K_i(theta') Linv_i^T.
#include "common.cuh"
#include "kernels_decl.h"
#include "tridiag.h"

#include <algorithm>
#include <atomic>
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace nugpr {

static std::atomic<long long> g_launches{0};
void note_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

void smem_optin(const void* func) {
  static std::atomic<const void*> done[64];
  for (auto& d : done) {
    const void* v = d.load();
    if (v == func) return;
    if (v == nullptr) {
      int dev = 0, optin = 0;
      cudaGetDevice(&dev);
      cudaError_t e1 = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes at;
      memset(&at, 0, sizeof(at));
      cudaError_t e2 = cudaFuncGetAttributes(&at, func);
      cudaError_t e3 = cudaSuccess;
      if (e1 == cudaSuccess && e2 == cudaSuccess)
        e3 = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(at.sharedSizeBytes));
      // full shared-memory carveout: otherwise the driver may pick a smaller L1/smem split
      // that admits fewer CTAs per SM than the launch plan assumes
      if (e3 == cudaSuccess)
        e3 = cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  static_cast<int>(cudaSharedmemCarveoutMaxShared));
      if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
        fprintf(stderr, "[nugpr] smem opt-in failed: optin=%d static=%zu (%s / %s / %s)\n", optin,
                static_cast<size_t>(at.sharedSizeBytes), cudaGetErrorString(e1), cudaGetErrorString(e2),
                cudaGetErrorString(e3));
        return;
      }
      const void* expect = nullptr;
      d.compare_exchange_strong(expect, func);
      return;
    }
  }
}

bool debug_sync() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("NUGPR_DEBUG_SYNC"); v = (e && e[0] == '1') ? 1 : 0; }
  return v == 1;
}

void post_launch(const char* name) {
  if (!debug_sync()) return;
  cudaError_t e = cudaDeviceSynchronize();
  cudaError_t l = cudaPeekAtLastError();
  fprintf(stderr, "[nugpr] %-22s sync=%s last=%s\n", name, cudaGetErrorString(e), cudaGetErrorString(l));
}

// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// Assemble K_i(theta) = k(X_i, X_i) + (noise + jitter_i) I into dst (ld x ld col-major),
// padding = identity.  grid = (tiles32 x tiles32 of the largest block, #blocks in list).
struct AsmArgs {
  const double* X;       // n x d, cluster-sorted
  int d;
  const int64_t* off;
  const int64_t* boff;
  const int32_t* ld;
  const int32_t* list;   // NULL => blockIdx.y is the cluster
  const double* jitter;  // [n_c] or NULL
  double* dst;
  int kind;
  double lam, noise, alpha;
};

__global__ void __launch_bounds__(256) assemble_kernel(AsmArgs a) {
  const int i = a.list ? a.list[blockIdx.y] : blockIdx.y;
  const int ld = a.ld[i];
  const int nt = (ld + 31) / 32;
  const int tr = blockIdx.x % nt, tc = blockIdx.x / nt;
  if (tc >= nt) return;
  const int64_t o = a.off[i];
  const int b = static_cast<int>(a.off[i + 1] - o);
  __shared__ double xr[32 * 33], xc[32 * 33];
  const int d = a.d;
  for (int idx = threadIdx.x; idx < 32 * d; idx += blockDim.x) {
    int rr = idx / d, dd = idx % d;
    int r = tr * 32 + rr, c = tc * 32 + rr;
    xr[rr * 33 + dd] = (r < b) ? a.X[(o + r) * d + dd] : 0.0;
    xc[rr * 33 + dd] = (c < b) ? a.X[(o + c) * d + dd] : 0.0;
  }
  __syncthreads();
  const double diag_add = a.noise + (a.jitter ? a.jitter[i] : 0.0);
  double* K = a.dst + a.boff[i];
  const int rr = threadIdx.x & 31;
  for (int cc = threadIdx.x >> 5; cc < 32; cc += 8) {
    const int r = tr * 32 + rr, c = tc * 32 + cc;
    if (r >= ld || c >= ld) continue;
    double v;
    if (r < b && c < b) {
      double sq = 0.0;
      for (int dd = 0; dd < d; ++dd) {
        double df = __dsub_rn(xr[rr * 33 + dd], xc[cc * 33 + dd]);
        sq = __dadd_rn(sq, __dmul_rn(df, df));
      }
      v = kval(a.kind, sq, a.lam, a.alpha);
      if (r == c) v += diag_add;
    } else {
      v = (r == c) ? 1.0 : 0.0;
    }
    K[static_cast<int64_t>(c) * ld + r] = v;
  }
}

void launch_assemble(const double* X, int d, const LayoutDev& L, const int32_t* list, int nlist,
                     int ld_max, const double* jitter, double* dst, int kind, double lam,
                     double noise, double alpha, cudaStream_t s) {
  AsmArgs a{X, d, L.off, L.boff, L.ld, list, jitter, dst, kind, lam, noise, alpha};
  int nt = (ld_max + 31) / 32;
  dim3 grid(nt * nt, list ? nlist : L.n_c);
  assemble_kernel<<<grid, 256, 0, s>>>(a);
  note_launch(); post_launch("assemble_kernel");
}

// ---------------------------------------------------------------------------------------
// Batched Cholesky + triangular inverse, one CTA per cluster, in place.
// Right-looking blocked Cholesky with 32-column panels staged in shared memory:
//   for each panel: load A[k0:ld, k0:k0+nb] -> smem, unblocked factorisation of the tall
//   panel (column scale + in-panel rank-1 updates), write back, then trailing update
//   A[k0+nb:, k0+nb:] -= P P^T (lower triangle) from smem.
// Then Linv = L^{-1} by tile rows:  X_II = L_II^{-1};  X_I,0:I0 = -X_II (L_I,0:I0 X_0:I0,0:I0).
// Also: status (0 ok / 1 not SPD), logdet partial 2 sum log L_jj, u = Linv 1_b.
constexpr int NB = 32;

struct CholArgs {
  double* A;             // block storage (in: K, out: Linv)
  const int64_t* off;
  const int64_t* poff;
  const int64_t* boff;
  const int32_t* ld;
  const int32_t* list;
  int32_t* status;       // [n_c]
  double* logdet_blk;    // [n_c]
  double* u;             // [n_pad]
};

__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int PR_T>   // panel rows per thread: ld <= PR_T * NT
__global__ void __launch_bounds__(256, (PR_T == 1) ? 2 : 1) chol_trtri_kernel(CholArgs a) {
  const int i = a.list ? a.list[blockIdx.x] : blockIdx.x;
  const int ld = a.ld[i];
  const int b = static_cast<int>(a.off[i + 1] - a.off[i]);
  double* A = a.A + a.boff[i];
  extern __shared__ double sm[];
  __shared__ int fail;
  __shared__ double red[8];
  const int tid = threadIdx.x;
  if (tid == 0) fail = 0;
  __syncthreads();

  // ---------------- Cholesky (right-looking, NB-column panels) ----------------
  // Panel Pn is column-major in smem with leading dimension pr (rows contiguous): every
  // per-row sweep is unit-stride across lanes (no bank conflicts).
  double* Pn = sm;
  for (int k0 = 0; k0 < ld; k0 += NB) {
    const int nb = min(NB, ld - k0);
    const int pr = ld - k0;          // panel rows
    // Panel factorisation with the panel rows in REGISTERS: thread t owns panel rows t, t + NT, ...
    // (PR_T rows of 32 columns).  Column step j costs ONE barrier: before it, the owner of row j
    // publishes the pivot d_j = sqrt(a_jj) and every top-row owner (r < 32) its current a_rj; after
    // it, each thread scales its own a_rj by 1/d_j and updates its row with the top rows' a_cj / d_j
    // formed on the fly (the same roundings as scaling the column first).
    double prow[PR_T][NB];
#pragma unroll
    for (int h = 0; h < PR_T; ++h) {
      const int r = tid + h * NT;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        prow[h][c] = (r < pr && c < nb) ? A[static_cast<int64_t>(k0 + c) * ld + k0 + r] : 0.0;
    }
    __shared__ double lcol[2][NB], dpiv[NB];
    if (tid < NB) {
      lcol[0][tid] = prow[0][0];                          // column 0 of the top rows
      if (tid == 0) {
        const double piv = prow[0][0];
        if (!(piv > 0.0)) fail = 1;
        dpiv[0] = sqrt(piv > 0.0 ? piv : 1.0);
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      if (j < nb) {
        const double dgv = dpiv[j];
        const double inv = 1.0 / dgv;
        const double* uc = lcol[j & 1];
#pragma unroll
        for (int h = 0; h < PR_T; ++h) {
          const int r = tid + h * NT;
          if (r > j && r < pr) {
            const double l = prow[h][j] * inv;
            prow[h][j] = l;
#pragma unroll
            for (int c = j + 1; c < NB; ++c)
              if (c <= r) prow[h][c] -= l * (uc[c] * inv);
          } else if (r == j) {
            prow[h][j] = dgv;
          }
        }
        if (j + 1 < nb) {
          // publish column j+1 of the top rows and its pivot for the next step
#pragma unroll
          for (int h = 0; h < PR_T; ++h) {
            const int r = tid + h * NT;
            if (r < NB) lcol[(j + 1) & 1][r] = prow[h][j + 1];
            if (r == j + 1) {
              const double piv = prow[h][j + 1];
              if (!(piv > 0.0)) fail = 1;
              dpiv[j + 1] = sqrt(piv > 0.0 ? piv : 1.0);
            }
          }
          __syncthreads();
        }
      }
    }
    // the finished panel to shared memory (the trailing update reads it) and global
#pragma unroll
    for (int h = 0; h < PR_T; ++h) {
      const int r = tid + h * NT;
      if (r < pr)
#pragma unroll
        for (int c = 0; c < NB; ++c) Pn[c * pr + r] = (c < nb && r >= c) ? prow[h][c] : 0.0;
    }
    __syncthreads();
    for (int idx = tid; idx < pr * nb; idx += NT) {
      const int c = idx / pr, r = idx % pr;
      A[static_cast<int64_t>(k0 + c) * ld + k0 + r] = (r >= c) ? Pn[c * pr + r] : 0.0;
    }
    // trailing update of the lower triangle: A[t+r][t+c] -= sum_j P[nb+r][j] P[nb+c][j], r >= c,
    // in 64x64 output tiles, 4x4 register tile per thread, coalesced read-modify-write of A.
    const int tr = pr - nb;
    if (tr > 0) {
      const int t0 = k0 + nb;
      const int nt = (tr + 63) / 64;
      const int ntl = nt * (nt + 1) / 2;
      // FP64 DMMA: 8 warps as 2 x 4, warp tile 32 x 16 of each 64x64 output tile, K = nb panel columns
      const int lane = tid & 31, wid = tid >> 5, wm = wid & 1, wn = wid >> 1;
      const int qr = lane >> 2, qc = lane & 3;
      for (int tt = 0; tt < ntl; ++tt) {
        int bi = static_cast<int>((sqrt(8.0 * tt + 1.0) - 1.0) * 0.5);
        while (bi * (bi + 1) / 2 > tt) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= tt) ++bi;
        const int bj = tt - bi * (bi + 1) / 2;
        const int rw = bi * 64 + wm * 32, cw = bj * 64 + wn * 16;   // warp tile origin (trailing block)
        double acc[4][2][2];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int n = 0; n < 2; ++n) { acc[m][n][0] = 0.0; acc[m][n][1] = 0.0; }
        if (rw < tr && cw < tr && rw + 31 >= cw) {
          for (int k4 = 0; k4 < nb; k4 += 4) {
            const double* pk = Pn + (k4 + qc) * pr + nb;            // panel column k4+qc, trailing rows
            double af[4], bf[2];
#pragma unroll
            for (int m = 0; m < 4; ++m) { const int r = rw + m * 8 + qr; af[m] = (r < tr) ? pk[r] : 0.0; }
#pragma unroll
            for (int n = 0; n < 2; ++n) { const int c = cw + n * 8 + qr; bf[n] = (c < tr) ? pk[c] : 0.0; }
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
              for (int n = 0; n < 2; ++n) dmma_c(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
          }
          // read-modify-write of the trailing tile: all 16 loads in flight, then the stores
          double old_[4][2][2];
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int r = rw + m * 8 + qr, c = cw + n * 8 + 2 * qc + e;
                old_[m][n][e] = (r < tr && c < tr && r >= c) ? A[static_cast<int64_t>(t0 + c) * ld + t0 + r] : 0.0;
              }
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int r = rw + m * 8 + qr, c = cw + n * 8 + 2 * qc + e;
                if (r < tr && c < tr && r >= c) A[static_cast<int64_t>(t0 + c) * ld + t0 + r] = old_[m][n][e] - acc[m][n][e];
              }
        }
      }
    }
    __syncthreads();
  }
  // logdet partial (real rows only; padding diagonal is 1)
  double ls = 0.0;
  for (int r = tid; r < b; r += NT) ls += log(A[static_cast<int64_t>(r) * ld + r]);
  ls = warp_sum(ls);
  if ((tid & 31) == 0) red[tid >> 5] = ls;
  __syncthreads();
  if (tid == 0) {
    double s_ = 0.0;
    for (int w = 0; w < NT / 32; ++w) s_ += red[w];
    a.logdet_blk[i] = 2.0 * s_;
    a.status[i] = fail;
  }
  __syncthreads();
  if (fail) return;

  // ---------------- triangular inverse (in place, by row panels) ----------------
  // Row panel I = rows [I0, I0+nb).  smem (all column-major: rows contiguous):
  //   LrT[k*NB + r] = L[I0+r][k] (k < I0+nb),  XdT[k*NB + r] = (L_II^{-1})[r][k],
  //   Yc[cl*NB + r] = (L[I,0:I0] * Xinv[0:I0, cc0+cl])[r].
  constexpr int YC = 64;
  constexpr int NBP = NB + 1;                 // padded stride: conflict-free column sweeps
  constexpr int XKC = 32, XSP = YC + 4;       // staged X rows per chunk; row stride (conflict-free B fragments)
  double* LrT = sm;
  for (int I0 = 0; I0 < ld; I0 += NB) {
    const int nb = min(NB, ld - I0);
    const int ldr = I0 + nb;
    double* XdT = LrT + NBP * ldr;            // NB x NB (stride NBP)
    double* Yc = XdT + NBP * NB;              // NB x YC
    double* Xs = Yc + NB * YC;                // XKC x XSP
    for (int idx = tid; idx < nb * ldr; idx += NT) {
      const int k = idx / nb, r = idx % nb;   // coalesced over r in global and smem
      LrT[k * NBP + r] = A[static_cast<int64_t>(k) * ld + I0 + r];
    }
    __syncthreads();
    // diagonal tile inverse: thread j < nb solves L_II x = e_j by forward substitution
    if (tid < nb) {
      // column j of L_II^{-1} by forward substitution, kept in registers (fully unrolled)
      const int j = tid;
      double x[NB];
#pragma unroll
      for (int r = 0; r < NB; ++r) {
        double v = 0.0;
        if (r < nb && r >= j) {
          v = (r == j) ? 1.0 : 0.0;
#pragma unroll
          for (int k = 0; k < r; ++k)
            if (k >= j) v -= LrT[(I0 + k) * NBP + r] * x[k];
          v *= 1.0 / LrT[(I0 + r) * NBP + r];
        }
        x[r] = v;
      }
#pragma unroll
      for (int r = 0; r < NB; ++r) XdT[j * NBP + r] = x[r];     // column j of the inverse
    }
    __syncthreads();
    for (int cc0 = 0; cc0 < I0; cc0 += YC) {
      const int ncc = min(YC, I0 - cc0);
      // Y = L[I, c..I0) X[c..I0, cc0:cc0+64) and X[I, cc0:..] = -Xd Y, both on the FP64 tensor
      // pipe: warp w owns the 8 columns cc0 + 8w.. (one n8 tile) and the 4 m8 tiles of the 32 rows
      {
        const int lane = tid & 31, wid = tid >> 5;
        const int qr = lane >> 2, qc = lane & 3;
        const int c8 = wid * 8;                               // column offset within the block
        double acc[4][2];
#pragma unroll
        for (int m = 0; m < 4; ++m) { acc[m][0] = 0.0; acc[m][1] = 0.0; }
        // X[k][cc0 : cc0+64] staged through shared memory 32 rows at a time (coalesced column runs)
        // instead of per-fragment global loads inside the tensor loop
        for (int kc = cc0; kc < I0; kc += XKC) {
          const int nk = min(XKC, I0 - kc);
          for (int idx = tid; idx < nk * YC; idx += NT) {
            const int cl = idx / nk, kl = idx - cl * nk;
            Xs[kl * XSP + cl] = (cl < ncc) ? A[static_cast<int64_t>(cc0 + cl) * ld + kc + kl] : 0.0;
          }
          __syncthreads();
          if (c8 < ncc) {
            // X is lower triangular: rows k < cc0 + c8 of these columns are zero
            const int kstart = max(kc, cc0 + c8);
            for (int k4 = kstart; k4 < kc + nk; k4 += 4) {
              const double bf = Xs[(k4 - kc + qc) * XSP + c8 + qr];
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                const int r = m * 8 + qr;
                const double af = (r < nb) ? LrT[(k4 + qc) * NBP + r] : 0.0;
                dmma_c(acc[m][0], acc[m][1], af, bf);
              }
            }
          }
          __syncthreads();
        }
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int e = 0; e < 2; ++e) Yc[(c8 + 2 * qc + e) * NB + m * 8 + qr] = acc[m][e];
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 4; ++m) { acc[m][0] = 0.0; acc[m][1] = 0.0; }
        if (c8 < ncc) {
          for (int k4 = 0; k4 < nb; k4 += 4) {
            const double bf = Yc[(c8 + qr) * NB + k4 + qc];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const int r = m * 8 + qr;
              const double af = (r < nb) ? XdT[(k4 + qc) * NBP + r] : 0.0;
              dmma_c(acc[m][0], acc[m][1], af, bf);
            }
          }
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int r = m * 8 + qr, cl = c8 + 2 * qc + e;
              if (r < nb && cl < ncc) A[static_cast<int64_t>(cc0 + cl) * ld + I0 + r] = -acc[m][e];
            }
        }
        __syncthreads();
      }
    }
    for (int idx = tid; idx < nb * nb; idx += NT) {
      const int r = idx % nb, c = idx / nb;
      A[static_cast<int64_t>(I0 + c) * ld + I0 + r] = (r >= c) ? XdT[c * NBP + r] : 0.0;
    }
    // strict upper triangle right of the diagonal tile := 0
    for (int idx = tid; idx < nb * (ld - I0 - nb); idx += NT) {
      const int r = idx % nb, c = I0 + nb + idx / nb;
      A[static_cast<int64_t>(c) * ld + I0 + r] = 0.0;
    }
    __syncthreads();
  }
  // u = Linv * 1_b  (row sums over the real columns); rows >= b are padding => 0
  const int64_t p0 = a.poff[i];
  for (int r = tid; r < ld; r += NT) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (r < b) {
      int k = 0;
      for (; k + 3 <= r; k += 4) {
        a0 += A[static_cast<int64_t>(k) * ld + r];
        a1 += A[static_cast<int64_t>(k + 1) * ld + r];
        a2 += A[static_cast<int64_t>(k + 2) * ld + r];
        a3 += A[static_cast<int64_t>(k + 3) * ld + r];
      }
      for (; k <= r; ++k) a0 += A[static_cast<int64_t>(k) * ld + r];
    }
    a.u[p0 + r] = (a0 + a1) + (a2 + a3);
  }
}

size_t chol_smem_bytes(int ld_max) {
  size_t panel = static_cast<size_t>(ld_max) * NB;                         // Cholesky panel
  size_t inv = static_cast<size_t>(NB + 1) * ld_max + (NB + 1) * NB + static_cast<size_t>(NB) * 64 + 32 * 68 + 64;
  return sizeof(double) * (panel > inv ? panel : inv);
}

void launch_chol_trtri(double* A, const LayoutDev& L, const int32_t* list, int nlist, int ld_max,
                       int32_t* status, double* logdet_blk, double* u, cudaStream_t s) {
  CholArgs a{A, L.off, L.poff, L.boff, L.ld, list, status, logdet_blk, u};
  size_t smem = chol_smem_bytes(ld_max);
  if (ld_max <= NT) {
    smem_optin(reinterpret_cast<const void*>(chol_trtri_kernel<1>));
    chol_trtri_kernel<1><<<list ? nlist : L.n_c, NT, smem, s>>>(a);
  } else {
    smem_optin(reinterpret_cast<const void*>(chol_trtri_kernel<2>));
    chol_trtri_kernel<2><<<list ? nlist : L.n_c, NT, smem, s>>>(a);
  }
  note_launch(); post_launch("chol_trtri_kernel");
}

// ---------------------------------------------------------------------------------------
// Batched FP64 GEMM on cluster blocks: C_i = A_i * op(B_i), all ld_i x ld_i col-major.
//   op(B)(k,c) = TRANSB ? B[k*ld + c] (= B^T) : B[c*ld + k]
//   A_LOWER: A(r,k) = 0 for k > r;  B_LOWERT: op(B)(k,c) = 0 for k > c (B^T of a lower matrix)
//   SYM: C symmetric — only tiles with tile_r >= tile_c are computed and mirrored.
struct GemmArgs {
  const double* A;
  const double* B;
  double* C;
  const int64_t* boff;
  const int32_t* ld;
  int ntile_max;         // tiles per dimension of the largest block
  const int64_t* pboff;  // PACKED output: C_i's packed lower-tile storage at pboff[i] (else NULL)
};

// Batched block GEMM on the FP64 tensor pipe (mma.sync m8n8k4 f64).  64x64 CTA tile, 8 warps as 2 (rows) x 4 (cols), warp tile 32x16 =
// 4 x 2 m8n8 tiles; K staged 16 at a time in shared memory (k-major, row stride 68 = 4 mod 16
// so the fragment loads are bank-conflict free), register double buffering of the next stage.
// 8x8 sub-tiles entirely outside the block (ld is a multiple of 8) are skipped.
constexpr int GLD = 68;

// (not volatile: a pure function of its operands, so the compiler may interleave it with the loads)
__device__ __forceinline__ void dmma884g(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <bool TRANSB, bool A_LOWER, bool B_LOWERT, bool SYM, bool PACKED>
__global__ void __launch_bounds__(256, 3) gemm_dmma_kernel(GemmArgs g) {
  const int i = blockIdx.y;
  const int ld = g.ld[i];
  const int nt = (ld + 63) / 64;
  int tr, tc;
  if (SYM) {
    int t = blockIdx.x;
    if (t >= nt * (nt + 1) / 2) return;
    tr = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (tr * (tr + 1) / 2 > t) --tr;
    while ((tr + 1) * (tr + 2) / 2 <= t) ++tr;
    tc = t - tr * (tr + 1) / 2;
  } else {
    if (static_cast<int>(blockIdx.x) >= nt * nt) return;
    tr = blockIdx.x % nt;
    tc = blockIdx.x / nt;
  }
  const int64_t bo = g.boff[i];
  const double* A = g.A + bo;
  const double* B = g.B + bo;
  double* C = g.C + (PACKED ? g.pboff[i] : bo);
  const int r0 = tr * 64, c0 = tc * 64;
  int kend = ld;
  if (A_LOWER) kend = min(kend, r0 + 64);
  if (B_LOWERT) kend = min(kend, c0 + 64);
  __shared__ __align__(16) double As[2][16 * GLD];
  __shared__ __align__(16) double Bs[2][16 * GLD];
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int wm = wid & 1, wn = wid >> 1;
  const int qr = lane >> 2, qc = lane & 3;
  // global -> register staging: 4 A and 4 B values per thread per stage
  double ra[4], rb[4];
  auto gload = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + u * 256;
      {
        const int kk = idx >> 6, rr = idx & 63;
        const int r = r0 + rr, k = k0 + kk;
        ra[u] = (r < ld && k < ld) ? A[static_cast<int64_t>(k) * ld + r] : 0.0;
      }
      {
        int kk, cc;
        if (TRANSB) { kk = idx >> 6; cc = idx & 63; }
        else        { cc = idx >> 4; kk = idx & 15; }
        const int c = c0 + cc, k = k0 + kk;
        double v = 0.0;
        if (c < ld && k < ld) v = TRANSB ? B[static_cast<int64_t>(k) * ld + c] : B[static_cast<int64_t>(c) * ld + k];
        rb[u] = v;
      }
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + u * 256;
      As[buf][(idx >> 6) * GLD + (idx & 63)] = ra[u];
      if (TRANSB) Bs[buf][(idx >> 6) * GLD + (idx & 63)] = rb[u];
      else        Bs[buf][(idx & 15) * GLD + (idx >> 4)] = rb[u];
    }
  };
  double acc[4][2][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) { acc[m][n][0] = 0.0; acc[m][n][1] = 0.0; }
  // which 8x8 sub-tiles of this warp lie inside the block
  const int wr = r0 + wm * 32, wc = c0 + wn * 16;
  const int mval = max(0, min(4, (ld - wr) >> 3));
  const int nval = max(0, min(2, (ld - wc) >> 3));
  if (kend > 0) {
    gload(0);
    sstore(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < kend; k0 += 16) {
      const bool more = k0 + 16 < kend;
      if (more) gload(k0 + 16);
      const double* as = As[buf];
      const double* bs = Bs[buf];
#pragma unroll
      for (int k4 = 0; k4 < 16; k4 += 4) {
        double af[4], bf[2];
#pragma unroll
        for (int m = 0; m < 4; ++m) af[m] = as[(k4 + qc) * GLD + wm * 32 + m * 8 + qr];
#pragma unroll
        for (int n = 0; n < 2; ++n) bf[n] = bs[(k4 + qc) * GLD + wn * 16 + n * 8 + qr];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int n = 0; n < 2; ++n)
            if (m < mval && n < nval) dmma884g(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
      }
      if (more) {
        sstore(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
  // C fragment: row qr, columns 2qc, 2qc+1 of each 8x8 tile
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      if (m >= mval || n >= nval) continue;
      const int r = wr + m * 8 + qr;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = wc + n * 8 + 2 * qc + e;
        const double v = acc[m][n][e];
        if (PACKED) {
          // lower tiles (r/8 >= c/8) in the packed block order, swizzled (common.cuh); the diagonal
          // tiles are written from their lower half and mirrored, so they are exactly symmetric
          const int I = r >> 3, K = c >> 3, mt = ld >> 3;
          if (r >= c) {
            double* tp = C + static_cast<int64_t>(pk_tile(I, K, mt)) * 64;
            tp[swz(r & 7, c & 7)] = v;
            if (I == K) tp[swz(c & 7, r & 7)] = v;
          }
        } else if (SYM) {
          if (r >= c) {
            C[static_cast<int64_t>(c) * ld + r] = v;
            C[static_cast<int64_t>(r) * ld + c] = v;
          }
        } else {
          C[static_cast<int64_t>(c) * ld + r] = v;
        }
      }
    }
}

// H = Linv * Linv^T (symmetric)
void launch_gemm_H(const double* Linv, double* H, const LayoutDev& L, int ld_max, bool packed, cudaStream_t s) {
  int nt = (ld_max + 63) / 64;
  GemmArgs g{Linv, Linv, H, L.boff, L.ld, nt, L.pboff};
  if (packed) gemm_dmma_kernel<true, true, true, true, true><<<dim3(nt * (nt + 1) / 2, L.n_c), 256, 0, s>>>(g);
  else gemm_dmma_kernel<true, true, true, true, false><<<dim3(nt * (nt + 1) / 2, L.n_c), 256, 0, s>>>(g);
  note_launch(); post_launch("gemm_H");
}
// T = K * Linv^T
void launch_gemm_KLt(const double* K, const double* Linv, double* T, const LayoutDev& L, int ld_max,
                     cudaStream_t s) {
  int nt = (ld_max + 63) / 64;
  GemmArgs g{K, Linv, T, L.boff, L.ld, nt, nullptr};
  gemm_dmma_kernel<true, false, true, false, false><<<dim3(nt * nt, L.n_c), 256, 0, s>>>(g);
  note_launch(); post_launch("gemm_KLt");
}
// G = Linv * T (symmetric)
void launch_gemm_LT(const double* Linv, const double* T, double* G, const LayoutDev& L, int ld_max, bool packed,
                    cudaStream_t s) {
  int nt = (ld_max + 63) / 64;
  GemmArgs g{Linv, T, G, L.boff, L.ld, nt, L.pboff};
  if (packed) gemm_dmma_kernel<false, true, false, true, true><<<dim3(nt * (nt + 1) / 2, L.n_c), 256, 0, s>>>(g);
  else gemm_dmma_kernel<false, true, false, true, false><<<dim3(nt * (nt + 1) / 2, L.n_c), 256, 0, s>>>(g);
  note_launch(); post_launch("gemm_LT");
}

// ---------------------------------------------------------------------------------------
// Fixed-order sum of n doubles (single CTA) -> out[0].
__global__ void sum_kernel(const double* v, int n, double* out) {
  __shared__ double red[NT];
  double s = 0.0;
  const int per = (n + NT - 1) / NT;
  const int lo = threadIdx.x * per, hi = min(n, lo + per);
  for (int k = lo; k < hi; ++k) s += v[k];
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < NT; ++k) t += red[k];
    out[0] = t;
  }
}
void launch_sum(const double* v, int n, double* out, cudaStream_t s) {
  sum_kernel<<<1, NT, 0, s>>>(v, n, out);
  note_launch(); post_launch("sum_kernel");
}

// ---------------------------------------------------------------------------------------
// K_rep(theta) = k(r_i, r_j) (no noise, Eq. 22 / SPEC.md:74), n_c x n_c row-major.
__global__ void krep_kernel(const double* reps, int n_c, int d, int kind, double lam, double alpha,
                            double* K) {
  int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(n_c) * n_c) return;
  int r = static_cast<int>(idx / n_c), c = static_cast<int>(idx % n_c);
  double sq = 0.0;
  for (int dd = 0; dd < d; ++dd) {
    double df = __dsub_rn(reps[r * d + dd], reps[c * d + dd]);
    sq = __dadd_rn(sq, __dmul_rn(df, df));
  }
  K[idx] = kval(kind, sq, lam, alpha);
}
void launch_krep(const double* reps, int n_c, int d, int kind, double lam, double alpha, double* K,
                 cudaStream_t s) {
  int64_t tot = static_cast<int64_t>(n_c) * n_c;
  krep_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(reps, n_c, d, kind, lam, alpha, K);
  note_launch(); post_launch("krep_kernel");
}

// ---------------------------------------------------------------------------------------
// lambda_0 = lambda_min(K_rep) (Eq. 26) by Lanczos with full reorthogonalisation (two passes
// of classical Gram-Schmidt), run by ONE thread-block cluster of CS CTAs: CTA q owns rows
// [q*R, (q+1)*R) of K_rep (cached in its shared memory when they fit) and of every Lanczos
// vector; the per-iteration dot products are reduced across the cluster through distributed
// shared memory in fixed rank order, so every CTA holds bit-identical alpha/beta and takes
// the same convergence decision.  Converged when the Ritz residual beta_{k+1}|s_k| <=
// tol_rel*||K||_inf (then |theta - lambda| <= that bound).  Writes lam0, the normalised Ritz
// vector v0 (warm start of the next solve) and M = K - lam0 I.
struct LanczosArgs {
  const double* K;       // n_c x n_c row-major
  int n_c;
  const double* vinit;   // NULL or n_c
  double* V;             // (kmax+1) x n_c
  int kmax;
  double tol_rel;
  double* lam0;          // [1]
  double* v0;            // [n_c] out
  double* M;             // n_c x n_c out (K - lam0 I)
  int32_t* info;         // [3] {iterations, converged, lambda_0 not certifiably > 0}
  int cacheK;
  int kcache;            // Lanczos vectors cached in shared memory
};

constexpr int LZ_NT = 512;

// Number of eigenvalues of T (diag a, off b) below x, division-free: signs of the leading
// principal minors p_i = (a_i - x) p_{i-1} - b_{i-1}^2 p_{i-2}, rescaled by powers of two.
__device__ __forceinline__ int sturm_count_nodiv(int k, const double* a, const double* b, double x) {
  // p_0 = 1, p_1 = a_0 - x, p_{i+1} = (a_i - x) p_i - b_{i-1}^2 p_{i-1}; #sign changes = #eig < x.
  // A zero minor is replaced by a tiny value of the opposite sign of its predecessor.
  double pm2 = 1.0, pm1 = a[0] - x;
  if (pm1 == 0.0) pm1 = -1e-300;
  int cnt = (pm1 < 0.0) ? 1 : 0;
  for (int i = 1; i < k; ++i) {
    double p = (a[i] - x) * pm1 - b[i - 1] * b[i - 1] * pm2;
    if (p == 0.0) p = (pm1 > 0.0) ? -1e-300 : 1e-300;
    if ((p < 0.0) != (pm1 < 0.0)) ++cnt;
    const double ap = fabs(p);
    if (ap > 1e150 || ap < 1e-150) {
      const int e = ilogb(ap);
      pm1 = scalbn(pm1, -e);
      p = scalbn(p, -e);
    }
    pm2 = pm1;
    pm1 = p;
  }
  return cnt;
}

// smallest eigenvalue of the k x k tridiagonal (a, b) by LZ_NT-way multisection over the whole
// CTA (9+ bits per round); every thread returns the same value.
__device__ double block_tridiag_min_eig(int k, const double* a, const double* b, double hi_hint,
                                        int* cnt_sm, double* lohi) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    double lo = a[0], hi = a[0];
    for (int i = 0; i < k; ++i) {
      double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < k - 1 ? fabs(b[i]) : 0.0);
      lo = fmin(lo, a[i] - r);
      hi = fmax(hi, a[i] + r);
    }
    if (hi_hint < hi && sturm_count_nodiv(k, a, b, hi_hint) >= 1) hi = hi_hint;
    lohi[0] = lo;
    lohi[1] = hi;
  }
  __syncthreads();
  double lo = lohi[0], hi = lohi[1];
  (void)cnt_sm;
  for (int it = 0; it < 8; ++it) {
    if (!(hi - lo > 1e-16 * fabs(hi))) break;       // uniform: all threads hold the same values
    const double x = lo + (hi - lo) * (tid + 1) / (LZ_NT + 1.0);
    // the flags "some eigenvalue below x" are monotone in tid, so the first set one is at index f =
    // the number of unset ones: one counting barrier instead of a serial scan
    const int f = __syncthreads_count(sturm_count_nodiv(k, a, b, x) < 1);
    const double nlo = lo + (hi - lo) * f / (LZ_NT + 1.0);
    const double nhi = (f < LZ_NT) ? lo + (hi - lo) * (f + 1) / (LZ_NT + 1.0) : hi;
    lo = nlo;
    hi = nhi;
  }
  return 0.5 * (lo + hi);
}

// eigenvector of T for eigenvalue th: two inverse-iteration steps (Thomas, one division per row)
__device__ void tridiag_eigvec_fast(int k, const double* a, const double* b, double th, double* s,
                                    double* w) {
  double scale = 0.0;
  for (int i = 0; i < k; ++i) scale = fmax(scale, fabs(a[i]) + (i < k - 1 ? fabs(b[i]) : 0.0));
  const double tiny = 1e-300 + 1e-15 * scale;
  for (int i = 0; i < k; ++i) s[i] = 1.0;
  double* cp = w;
  double* dp = w + k;
  for (int step = 0; step < 2; ++step) {
    double den = a[0] - th;
    if (fabs(den) < tiny) den = (den >= 0 ? tiny : -tiny);
    double inv = 1.0 / den;
    cp[0] = (k > 1 ? b[0] : 0.0) * inv;
    dp[0] = s[0] * inv;
    for (int i = 1; i < k; ++i) {
      den = (a[i] - th) - b[i - 1] * cp[i - 1];
      if (fabs(den) < tiny) den = (den >= 0 ? tiny : -tiny);
      inv = 1.0 / den;
      cp[i] = (i < k - 1 ? b[i] : 0.0) * inv;
      dp[i] = (s[i] - b[i - 1] * dp[i - 1]) * inv;
    }
    s[k - 1] = dp[k - 1];
    for (int i = k - 2; i >= 0; --i) s[i] = dp[i] - cp[i] * s[i + 1];
    double nrm = 0.0;
    for (int i = 0; i < k; ++i) nrm += s[i] * s[i];
    nrm = 1.0 / sqrt(nrm);
    for (int i = 0; i < k; ++i) s[i] *= nrm;
  }
}

template <int CS>
__global__ void __launch_bounds__(LZ_NT, 1) lanczos_cluster_kernel(LanczosArgs a) {
  namespace cgs = cooperative_groups;
  cgs::cluster_group cl = cgs::this_cluster();
  const int q = static_cast<int>(cl.block_rank());
  const int n = a.n_c;
  const int kmax = a.kmax;
  const int R = (n + CS - 1) / CS;
  const int r0 = min(n, q * R), r1 = min(n, r0 + R), nr = r1 - r0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = LZ_NT / 32;
  extern __shared__ __align__(16) double sm[];
  double* vfull = sm;                 // n
  double* wl = vfull + n;             // R
  double* hp = wl + R;                // 2 * (kmax+1)   (partial dots, double-buffered)
  double* hs = hp + 2 * (kmax + 1);   // kmax+1         (cluster-summed dots)
  double* nb = hs + (kmax + 1);       // 4              (partial norms / scalars)
  double* al = nb + 4;                // kmax
  double* be = al + kmax;             // kmax
  double* ta = be + kmax;             // kmax
  double* tb = ta + kmax;             // kmax
  double* sv = tb + kmax;             // kmax
  double* sw = sv + kmax;             // 2 kmax
  double* part = sw + 2 * kmax;       // nw * R       (per-warp partial updates)
  double* Kc = part + nw * R;         // R * n (if cached)
  double* Vc = Kc + (a.cacheK ? static_cast<size_t>(R) * n : 0);   // kcache * R (Lanczos vectors, rows of this CTA)
  const int kcache = a.kcache;
  __shared__ double red[32];
  __shared__ int s_done, s_conv;
  __shared__ double s_theta;
  const double* Kg = a.K;
  auto Krow = [&](int r) -> const double* {   // r local
    return a.cacheK ? Kc + static_cast<int64_t>(r) * n : Kg + static_cast<int64_t>(r0 + r) * n;
  };
  auto Vrow = [&](int j) -> const double* {   // rows of this CTA of Lanczos vector j
    return (j < kcache) ? Vc + static_cast<int64_t>(j) * R : a.V + static_cast<int64_t>(j) * n + r0;
  };
  auto block_sum = [&](double v) -> double {
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w];
    return t;
  };
  // Cross-CTA reductions of one value per CTA: warp 0 reads the CS remote slots (one per lane),
  // butterfly-sums them (the same fixed order in every CTA, so all CTAs get the same bits) and
  // broadcasts through shared memory -- instead of every thread reading every remote slot.
  __shared__ double s_bc[4];
  int bc_i = 0;
  auto remote_sum = [&](double* slot, bool is_max) -> double {
    const int bi = bc_i;
    bc_i = (bc_i + 1) & 3;
    if (wid == 0) {
      double v = (lane < CS) ? *cl.map_shared_rank(slot, lane) : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, w) : v + w;
      }
      if (lane == 0) s_bc[bi] = v;
    }
    __syncthreads();
    return s_bc[bi];
  };
  auto cluster_sum = [&](int slot, double v) -> double {
    if (tid == 0) nb[slot] = v;
    cl.sync();
    return remote_sum(nb + slot, false);
  };
  auto store_v = [&](int j, int r, double v) {   // V[j][r0+r]
    a.V[static_cast<int64_t>(j) * n + r0 + r] = v;
    if (j < kcache) Vc[static_cast<int64_t>(j) * R + r] = v;
  };
  if (a.cacheK)
    for (int64_t idx = tid; idx < static_cast<int64_t>(nr) * n; idx += LZ_NT)
      Kc[idx] = Kg[static_cast<int64_t>(r0) * n + idx];
  __syncthreads();
  double rmax = 0.0;
  for (int r = wid; r < nr; r += nw) {
    const double* kr = Krow(r);
    double s = 0.0;
    for (int c = lane; c < n; c += 32) s += fabs(kr[c]);
    rmax = fmax(rmax, warp_sum(s));
  }
  if (lane == 0) red[wid] = rmax;
  __syncthreads();
  if (tid == 0) { double m = 0.0; for (int w = 0; w < nw; ++w) m = fmax(m, red[w]); nb[2] = m; s_done = 0; s_conv = 0; }
  cl.sync();
  const double knorm = remote_sum(nb + 2, true);
  __shared__ int cnt_sm[LZ_NT];
  __shared__ double lohi[2];
  // v_0: unnormalised start slice in wl, its squared norm partial in nb[3]
  double ss = 0.0;
  for (int r = tid; r < nr; r += LZ_NT) {
    const int g = r0 + r;
    double v = a.vinit ? a.vinit[g] : probe_value(0x5eed1a2c5ull, 0, g) * (1.0 + 0.01 * (g % 7));
    wl[r] = v;
    ss += v * v;
  }
  ss = block_sum(ss);
  if (tid == 0) nb[3] = ss;
  cl.sync();
  int k_final = 0;
  double theta = 0.0, theta_prev = INFINITY;
  double bprev = 0.0;
  for (int k = 0; k < kmax; ++k) {
    // exchange: v_k = w_{k} / ||w_k|| assembled from every CTA's wl slice (DSMEM), norm from nb[3]
    const double nn = remote_sum(nb + 3, false);
    const double inv = 1.0 / sqrt(nn);
    for (int c = tid; c < n; c += LZ_NT) {
      const int p = c / R, rr = c - p * R;
      vfull[c] = cl.map_shared_rank(wl, p)[rr] * inv;
    }
    if (k > 0 && tid == 0) be[k - 1] = sqrt(nn);
    cl.sync();                                    // everyone done reading remote wl / nb[3]
    for (int r = tid; r < nr; r += LZ_NT) store_v(k, r, vfull[r0 + r]);
    __syncthreads();
    for (int r = wid; r < nr; r += nw) {
      const double* kr = Krow(r);
      double s_ = 0.0;
      for (int c = lane; c < n; c += 32) s_ += kr[c] * vfull[c];
      s_ = warp_sum(s_);
      if (lane == 0) wl[r] = s_;
    }
    __syncthreads();
    double alpha = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      double* hpp = hp + pass * (kmax + 1);
      for (int j = wid; j <= k; j += nw) {
        const double* vj = Vrow(j);
        double s_ = 0.0;
        for (int r = lane; r < nr; r += 32) s_ += vj[r] * wl[r];
        s_ = warp_sum(s_);
        if (lane == 0) hpp[j] = s_;
      }
      cl.sync();
      // hs[j] = sum over the CTAs of hpp[j]: 16 lanes per j (lane group reads the CS slots),
      // segmented butterfly over the group
      for (int base = 0; base < 16 * (k + 1); base += LZ_NT) {   // warp-uniform trip count
        const int t0 = base + tid;
        const int j = t0 >> 4, p = t0 & 15;
        double v = (j <= k && p < CS) ? cl.map_shared_rank(hpp, p)[j] : 0.0;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (p == 0 && j <= k) hs[j] = v;
      }
      __syncthreads();
      alpha += hs[k];
      for (int r = lane; r < nr; r += 32) {
        double t = 0.0;
        for (int j = wid; j <= k; j += nw) t = fma(hs[j], Vrow(j)[r], t);
        part[wid * R + r] = t;
      }
      __syncthreads();
      for (int r = tid; r < nr; r += LZ_NT) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += part[w * R + r];
        wl[r] -= t;
      }
      __syncthreads();
    }
    double s2 = 0.0;
    for (int r = tid; r < nr; r += LZ_NT) s2 += wl[r] * wl[r];
    s2 = block_sum(s2);
    if (tid == 0) { al[k] = alpha; nb[3] = s2; }
    cl.sync();                                    // partial norms + new wl visible cluster-wide
    const double nn2 = remote_sum(nb + 3, false);
    const double beta = sqrt(nn2);
    if (tid == 0) be[k] = beta;
    (void)bprev;
    const int kk = k + 1;
    const bool last = (kk == kmax) || (kk == n) || !(beta > 1e-300);
    if (last || (kk >= 16 && kk % 8 == 0)) {
      for (int t = tid; t < kk; t += LZ_NT) { ta[t] = al[t]; tb[t] = (t < k) ? be[t] : beta; }
      __syncthreads();
      const double th = block_tridiag_min_eig(kk, ta, tb, theta_prev, cnt_sm, lohi);
      if (tid == 0) {
        tridiag_eigvec_fast(kk, ta, tb, th, sv, sw);
        const double res = fabs(beta * sv[kk - 1]);
        s_theta = th;
        const bool ok = res <= a.tol_rel * knorm;
        if (ok || last) {
          s_done = 1;
          s_conv = ok || !(beta > 1e-300) || (kk == n);
        }
      }
      __syncthreads();
      theta = s_theta;
      theta_prev = theta;
    }
    if (s_done) { k_final = kk; cl.sync(); break; }
  }
  // Ritz vector (rows of this CTA), normalised over the cluster; M = K - theta I
  double s3 = 0.0;
  for (int r = tid; r < nr; r += LZ_NT) {
    double v = 0.0;
    for (int j = 0; j < k_final; ++j) v += Vrow(j)[r] * sv[j];
    wl[r] = v;
    s3 += v * v;
  }
  const double vn = sqrt(cluster_sum(2, block_sum(s3)));
  for (int r = tid; r < nr; r += LZ_NT) a.v0[r0 + r] = wl[r] / vn;
  for (int64_t idx = tid; idx < static_cast<int64_t>(nr) * n; idx += LZ_NT) {
    const int r = static_cast<int>(idx / n), c = static_cast<int>(idx % n);
    const int64_t g = static_cast<int64_t>(r0) * n + idx;
    a.M[g] = Krow(r)[c] - ((r0 + r) == c ? theta : 0.0);
  }
  // info[2]: lambda_0 is not certifiably positive — within the Ritz-residual bound tol_rel ||K||_inf of
  // zero (|theta - lambda| <= that bound), e.g. duplicate representatives (reading P27)
  if (q == 0 && tid == 0) {
    a.lam0[0] = theta;
    a.info[0] = k_final;
    a.info[1] = s_conv;
    a.info[2] = (theta > a.tol_rel * knorm) ? 0 : 1;
  }
  cl.sync();   // keep shared memory alive until every CTA is done reading remote slots
}

size_t lanczos_scratch_doubles(int n_c, int kmax) {
  return static_cast<size_t>(kmax + 1) * n_c + 64;
}

template <int CS>
static cudaError_t lanczos_launch_cs(const LanczosArgs& a0, cudaStream_t s) {
  LanczosArgs a = a0;
  const int n = a.n_c, kmax = a.kmax, R = (n + CS - 1) / CS;
  size_t base = static_cast<size_t>(n) + R + 3 * (kmax + 1) + 4 + 7 * static_cast<size_t>(kmax) +
                static_cast<size_t>(LZ_NT / 32) * R;
  size_t withK = base + static_cast<size_t>(R) * n;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  auto kern = lanczos_cluster_kernel<CS>;
  cudaFuncAttributes fa;
  memset(&fa, 0, sizeof(fa));
  cudaFuncGetAttributes(&fa, kern);
  const size_t limit = static_cast<size_t>(optin) - fa.sharedSizeBytes - 256;
  a.cacheK = (withK * sizeof(double) <= limit) ? 1 : 0;
  size_t used = a.cacheK ? withK : base;
  long room = static_cast<long>(limit / sizeof(double)) - static_cast<long>(used);
  a.kcache = static_cast<int>(std::max<long>(0, std::min<long>(kmax + 1, room / std::max(1, R))));
  used += static_cast<size_t>(a.kcache) * R;
  const size_t smem = used * sizeof(double);
  if (smem > limit) return cudaErrorInvalidValue;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(limit));
  if (CS > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, 1, 1);
  cfg.blockDim = dim3(LZ_NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t launch_lanczos(const double* K, int n_c, const double* vinit, double* scratch, int kmax,
                           double tol_rel, double* lam0, double* v0, double* M, int32_t* info,
                           cudaStream_t s) {
  LanczosArgs a;
  a.K = K; a.n_c = n_c; a.vinit = vinit; a.V = scratch; a.kmax = kmax; a.tol_rel = tol_rel;
  a.lam0 = lam0; a.v0 = v0; a.M = M; a.info = info; a.cacheK = 0; a.kcache = 0;
  cudaError_t e;
  if (n_c >= 128) {
    e = lanczos_launch_cs<16>(a, s);
    if (e != cudaSuccess) { cudaGetLastError(); e = lanczos_launch_cs<8>(a, s); }
  } else {
    e = lanczos_launch_cs<4>(a, s);
  }
  note_launch(); post_launch("lanczos_cluster_kernel");
  return e;
}

}  // namespace nugpr
