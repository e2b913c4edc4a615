// cluster_kernels.cu — row A0 of SURVEY §8(a): Lloyd k-means on the training inputs
// ("k-means to find n_c clusters"), the stable sort of the points by cluster
// (the points of a cluster are stored contiguously) and the
// representatives (centroids; medoids, Eq. (32), reading P17).
//
// Reading P18 makes the assignment a deterministic function of the inputs:
//  * squared distances are summed in dimension order with separately rounded multiply and
//    add (__dmul_rn / __dadd_rn: no FMA contraction), ties go to the lowest centre index;
//  * centroid sums are exact int64 fixed-point sums (q = rint(x * 2^s)), accumulated with
//    integer atomics (associative, so the order in which CTAs arrive does not matter);
//  * the sort is a stable counting sort: per-chunk histograms, one exclusive scan in
//    (cluster, chunk) order, then an in-chunk stable rank.
// The only atomics of the library are the integer ones here.
#include <cstdint>

#include "common.cuh"
#include "kernels_decl.h"

namespace nugpr {

constexpr int KM_NT = 256;
constexpr int KM_CHUNK = 256;                // points per sort chunk (one CTA)
constexpr int KM_SMEM_CENTRES = 6144;        // centres (doubles) staged per CTA pass
constexpr int KM_SMEM_ACC = 4096;            // n_c*(d+1) limit for CTA-local accumulation
constexpr int KM_MQ = 128;                   // member tile of the medoid scores

// max |x| as the bit pattern of a non-negative double (monotone in the value).
__global__ void km_absmax_kernel(const double* X, int64_t cnt, unsigned long long* out) {
  double m = 0.0;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < cnt;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(X[k]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// Assignment step a(p) = argmin_j ||x_p - c_j||^2 fused with the fixed-point sums of the
// NEW assignment (the next update step's input) and the "changed" flag.
__global__ void __launch_bounds__(KM_NT) km_assign_kernel(const double* X, int64_t n, int d, int n_c,
                                                          const double* C, const int32_t* a_old,
                                                          int32_t* a_new, double scale,
                                                          unsigned long long* S, unsigned long long* cnt,
                                                          int32_t* changed) {
  extern __shared__ double kms[];
  const bool local_acc = n_c * (d + 1) <= KM_SMEM_ACC;
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(kms + KM_SMEM_CENTRES);
  if (local_acc)
    for (int k = threadIdx.x; k < n_c * (d + 1); k += blockDim.x) acc[k] = 0ull;
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool live = p < n;
  double x[32];
#pragma unroll
  for (int dd = 0; dd < 32; ++dd) x[dd] = (live && dd < d) ? X[p * d + dd] : 0.0;
  double best = __longlong_as_double(0x7ff0000000000000ll);   // +inf
  int arg = 0;
  const int per = max(1, KM_SMEM_CENTRES / d);
  for (int j0 = 0; j0 < n_c; j0 += per) {
    const int nj = min(per, n_c - j0);
    __syncthreads();
    for (int k = threadIdx.x; k < nj * d; k += blockDim.x) kms[k] = C[static_cast<int64_t>(j0) * d + k];
    __syncthreads();
    if (live) {
      for (int jj = 0; jj < nj; ++jj) {
        const double* c = kms + jj * d;
        double dist = 0.0;
#pragma unroll
        for (int dd = 0; dd < 32; ++dd) {
          if (dd < d) {
            const double df = __dsub_rn(x[dd], c[dd]);
            dist = __dadd_rn(dist, __dmul_rn(df, df));
          }
        }
        if (dist < best) { best = dist; arg = j0 + jj; }
      }
    }
  }
  __syncthreads();
  if (live) {
    a_new[p] = arg;
    if (a_old && a_old[p] != arg) *changed = 1;
    unsigned long long* dstS = local_acc ? acc : S;
    unsigned long long* dstC = local_acc ? acc + n_c * d : cnt;
#pragma unroll
    for (int dd = 0; dd < 32; ++dd)
      if (dd < d) {
        const long long q = __double2ll_rn(x[dd] * scale);      // exact scaling by 2^s, then RN-even
        atomicAdd(dstS + arg * d + dd, static_cast<unsigned long long>(q));
      }
    atomicAdd(dstC + arg, 1ull);
  }
  if (local_acc) {
    __syncthreads();
    for (int k = threadIdx.x; k < n_c * d; k += blockDim.x)
      if (acc[k]) atomicAdd(S + k, acc[k]);
    for (int k = threadIdx.x; k < n_c; k += blockDim.x)
      if (acc[n_c * d + k]) atomicAdd(cnt + k, acc[n_c * d + k]);
  }
}

// Update step: c_j = (double(S_j) * 2^-s) / count_j; empty clusters keep their centre.
// Zeroes the accumulators for the next assignment step.
__global__ void km_update_kernel(int n_c, int d, double inv_scale, unsigned long long* S,
                                 unsigned long long* cnt, double* C) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_c * d) return;
  const int j = k / d;
  const long long c = static_cast<long long>(cnt[j]);
  if (c > 0) {
    const double sum = static_cast<double>(static_cast<long long>(S[k]));
    C[k] = __ddiv_rn(__dmul_rn(sum, inv_scale), static_cast<double>(c));
  }
  S[k] = 0ull;
}
__global__ void km_zero_cnt_kernel(int n_c, unsigned long long* cnt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_c) cnt[k] = 0ull;
}

// Stable counting sort, pass 1: per-chunk histograms hist[j * n_chunks + chunk].
__global__ void __launch_bounds__(KM_CHUNK) km_hist_kernel(const int32_t* a, int64_t n, int n_c, int64_t n_chunks,
                                                           long long* hist) {
  extern __shared__ int hcnt[];
  for (int j = threadIdx.x; j < n_c; j += blockDim.x) hcnt[j] = 0;
  __syncthreads();
  const int64_t p = blockIdx.x * static_cast<int64_t>(KM_CHUNK) + threadIdx.x;
  if (p < n) atomicAdd(&hcnt[a[p]], 1);
  __syncthreads();
  for (int j = threadIdx.x; j < n_c; j += blockDim.x) hist[static_cast<int64_t>(j) * n_chunks + blockIdx.x] = hcnt[j];
}

// Pass 2: exclusive scan of hist (in place) by one CTA: each thread scans a contiguous
// segment, then the segment totals are scanned.
__global__ void __launch_bounds__(1024) km_scan_kernel(long long* v, int64_t len) {
  __shared__ long long tot[1024];
  const int64_t seg = (len + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * seg, e = min(len, b + seg);
  long long s = 0;
  for (int64_t k = b; k < e; ++k) s += v[k];
  tot[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int t = 0; t < static_cast<int>(blockDim.x); ++t) { long long x = tot[t]; tot[t] = run; run += x; }
  }
  __syncthreads();
  long long run = tot[threadIdx.x];
  for (int64_t k = b; k < e; ++k) { long long x = v[k]; v[k] = run; run += x; }
}

// Pass 3: stable scatter: rank = number of earlier points of the chunk in the same cluster.
__global__ void __launch_bounds__(KM_CHUNK) km_scatter_kernel(const int32_t* a, int64_t n, int64_t n_chunks,
                                                              const long long* base, int64_t* perm) {
  __shared__ int32_t ac[KM_CHUNK];
  const int64_t p0 = blockIdx.x * static_cast<int64_t>(KM_CHUNK);
  const int64_t p = p0 + threadIdx.x;
  ac[threadIdx.x] = (p < n) ? a[p] : -1;
  __syncthreads();
  if (p >= n) return;
  const int me = ac[threadIdx.x];
  int rank = 0;
  for (int q = 0; q < static_cast<int>(threadIdx.x); ++q) rank += (ac[q] == me);
  perm[base[static_cast<int64_t>(me) * n_chunks + blockIdx.x] + rank] = p;
}

// offsets[j] = base[j * n_chunks] (the first chunk's slot), offsets[n_c] = n.
__global__ void km_offsets_kernel(const long long* base, int n_c, int64_t n_chunks, int64_t n, int64_t* off) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n_c) off[j] = base[static_cast<int64_t>(j) * n_chunks];
  if (j == n_c) off[j] = n;
}

// dst[k, :] = src[idx[k], :] for k < rows (idx int64 or int32 via stride flag).
__global__ void km_gather_kernel(const double* src, int width, const int64_t* idx64, const int32_t* idx32,
                                 int64_t rows, double* dst) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= rows * width) return;
  const int64_t r = k / width, c = k % width;
  const int64_t s = idx64 ? idx64[r] : idx32[r];
  dst[k] = src[s * width + c];
}

// Medoid scores on cluster-sorted X: score_p = sum_{q in cluster(p)} k(x_p, x_q), q in order.
__global__ void __launch_bounds__(KM_NT) km_medoid_score_kernel(const double* Xs, int d, const int64_t* off,
                                                                int n_c, int kind, double lam, double alpha,
                                                                double* score) {
  const int j = blockIdx.y;
  const int64_t o = off[j], b = off[j + 1] - o;
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  __shared__ double xs[KM_MQ * 33];
  double x[32];
  const bool live = r < b;
#pragma unroll
  for (int dd = 0; dd < 32; ++dd) x[dd] = (live && dd < d) ? Xs[(o + r) * d + dd] : 0.0;
  double s = 0.0;
  for (int64_t q0 = 0; q0 < b; q0 += KM_MQ) {
    const int nq = static_cast<int>(b - q0 < KM_MQ ? b - q0 : KM_MQ);
    __syncthreads();
    for (int k = threadIdx.x; k < nq * d; k += blockDim.x) xs[(k / d) * 33 + k % d] = Xs[(o + q0) * d + k];
    __syncthreads();
    if (live) {
      for (int qq = 0; qq < nq; ++qq) {
        double sq = 0.0;
#pragma unroll
        for (int dd = 0; dd < 32; ++dd)
          if (dd < d) {
            const double df = __dsub_rn(x[dd], xs[qq * 33 + dd]);
            sq = __dadd_rn(sq, __dmul_rn(df, df));
          }
        s += kval(kind, sq, lam, alpha);
      }
    }
  }
  if (live) score[o + r] = s;
}

// Per-cluster argmax of the scores (first maximum in sorted order = lowest original index).
__global__ void __launch_bounds__(KM_NT) km_argmax_kernel(const double* score, const int64_t* off, int64_t* out) {
  const int j = blockIdx.x;
  const int64_t o = off[j], b = off[j + 1] - o;
  double bv = -__longlong_as_double(0x7ff0000000000000ll);
  int64_t bi = -1;
  for (int64_t r = threadIdx.x; r < b; r += blockDim.x) {
    const double v = score[o + r];
    if (v > bv) { bv = v; bi = r; }
  }
  __shared__ double sv[KM_NT];
  __shared__ int64_t si[KM_NT];
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int w = KM_NT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double v2 = sv[threadIdx.x + w];
      const int64_t i2 = si[threadIdx.x + w];
      if (i2 >= 0 && (si[threadIdx.x] < 0 || v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x]))) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = o + si[0];
}

// ------------------------------------------------------------------------------- launchers
void launch_km_absmax(const double* X, int64_t cnt, unsigned long long* out, cudaStream_t s) {
  const int grid = static_cast<int>((cnt + 255) / 256 + 1 < 1184 ? (cnt + 255) / 256 + 1 : 1184);
  km_absmax_kernel<<<grid, 256, 0, s>>>(X, cnt, out);
  note_launch(); post_launch("km_absmax_kernel");
}

size_t km_assign_smem() { return (KM_SMEM_CENTRES + KM_SMEM_ACC) * sizeof(double); }

void launch_km_assign(const double* X, int64_t n, int d, int n_c, const double* C, const int32_t* a_old,
                      int32_t* a_new, double scale, unsigned long long* S, unsigned long long* cnt,
                      int32_t* changed, cudaStream_t s) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(km_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(km_assign_smem()));
    init = true;
  }
  const int grid = static_cast<int>((n + KM_NT - 1) / KM_NT);
  km_assign_kernel<<<grid, KM_NT, km_assign_smem(), s>>>(X, n, d, n_c, C, a_old, a_new, scale, S, cnt, changed);
  note_launch(); post_launch("km_assign_kernel");
}

void launch_km_update(int n_c, int d, double inv_scale, unsigned long long* S, unsigned long long* cnt,
                      double* C, cudaStream_t s) {
  km_update_kernel<<<(n_c * d + 255) / 256, 256, 0, s>>>(n_c, d, inv_scale, S, cnt, C);
  km_zero_cnt_kernel<<<(n_c + 255) / 256, 256, 0, s>>>(n_c, cnt);
  note_launch(2); post_launch("km_update_kernel");
}

int64_t km_chunks(int64_t n) { return (n + KM_CHUNK - 1) / KM_CHUNK; }

void launch_km_sort(const int32_t* a, int64_t n, int n_c, long long* hist, int64_t* perm, int64_t* off,
                    cudaStream_t s) {
  const int64_t nch = km_chunks(n);
  const size_t hsm = sizeof(int) * static_cast<size_t>(n_c);
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(km_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    init = true;
  }
  km_hist_kernel<<<static_cast<unsigned>(nch), KM_CHUNK, hsm, s>>>(a, n, n_c, nch, hist);
  km_scan_kernel<<<1, 1024, 0, s>>>(hist, nch * n_c);
  km_scatter_kernel<<<static_cast<unsigned>(nch), KM_CHUNK, 0, s>>>(a, n, nch, hist, perm);
  km_offsets_kernel<<<(n_c + 1 + 255) / 256, 256, 0, s>>>(hist, n_c, nch, n, off);
  note_launch(4); post_launch("km_sort");
}

void launch_km_gather(const double* src, int width, const int64_t* idx64, const int32_t* idx32, int64_t rows,
                      double* dst, cudaStream_t s) {
  const int64_t tot = rows * width;
  if (tot == 0) return;
  km_gather_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(src, width, idx64, idx32, rows, dst);
  note_launch(); post_launch("km_gather_kernel");
}

void launch_km_medoids(const double* Xs, int d, const int64_t* off, int n_c, int64_t b_max, int kind, double lam,
                       double alpha, double* score, int64_t* out, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((b_max + KM_NT - 1) / KM_NT), n_c);
  km_medoid_score_kernel<<<grid, KM_NT, 0, s>>>(Xs, d, off, n_c, kind, lam, alpha, score);
  km_argmax_kernel<<<n_c, KM_NT, 0, s>>>(score, off, out);
  note_launch(2); post_launch("km_medoids");
}

}  // namespace nugpr
