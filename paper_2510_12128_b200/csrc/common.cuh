// common.cuh — device-side layout and state shared by the nuGPR kernels.
//
// Internal data layout in HBM:
//  * Clusters are padded to ld_i = round_up(b_i, 8) rows ("padded rows", reading P19); the
//    padding rows are identity rows in every block matrix and zero in every vector, so they
//    are exactly invisible to the method.
//  * Vectors: column-major [NC][n_pad] FP64 (one contiguous length-n_pad column per RHS;
//    column 0 = the y-solve, columns 1..m = the Hutchinson probes).
//  * Block matrices (Linv_i, H_i, G_i): dense ld_i x ld_i column-major at boff[i];
//    H and G are stored full (both triangles) so the apply streams them coalesced.
//  * Row tiles: a cluster is split into tiles of <= TILE_ROWS padded rows; each apply /
//    update CTA owns one tile; per-tile partial sums (S = W^T D partials, dots) live in
//    [n_tiles][16] arrays and are reduced in fixed tile order (deterministic).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nugpr {

constexpr int MAXC = 16;        // max columns per apply (1 + m)
constexpr int NT = 256;         // threads per CTA for the tile kernels
constexpr int TILE_ROWS = 512;  // max padded rows per tile (= whole clusters in this build)
constexpr int MAX_NSTAGE = 16;  // max TMA ring depth of the apply kernel
constexpr int SLOT_TARGET_DOUBLES = 4096;  // ~32 KB per TMA chunk
constexpr int PAD = 8;          // cluster padding granularity (rows)
constexpr int CTW = 16;         // columns per task of the DMMA column apply

struct TileDesc {
  int32_t blk;    // cluster index
  int32_t row0;   // first padded row within the cluster
  int32_t nrows;  // rows in this tile (even)
  int32_t pad_;
};

struct LayoutDev {
  const int64_t* off;    // [n_c+1] original (unpadded) row offsets
  const int64_t* poff;   // [n_c+1] padded row offsets
  const int64_t* boff;   // [n_c] element offset of block i in block storage
  const int32_t* ld;     // [n_c] padded cluster size
  const TileDesc* tiles; // [n_tiles]
  const int32_t* tile0;  // [n_c+1] tile range of each cluster
  const TileDesc* ctasks; // [n_ctasks] column tasks of the DMMA column apply: (cluster, col0, ncols)
  const int32_t* ctask0; // [n_c+1] column-task range of each cluster
  int32_t n_c;
  int32_t n_tiles;
  int32_t n_ctasks;
  int64_t n;             // unpadded rows
  int64_t n_pad;         // padded rows (vector column stride)
};

// Per-evaluation operator parameters (device resident so one captured graph serves all
// evaluation modes).  A D = a*D + b_i*B_i*D + u_i*(mscale * Mp S)_i with b_i = b0 + b1*jitter_i.
struct EvalParams {
  double a;
  double b0, b1;
  const double* B;       // H or G (block storage layout), NULL => no block term
  const float* B32;      // FP32-stored copy of B (NUGPR_F32_BLOCKS storage), NULL in FP64 mode
  const double* Mp;      // n_c x n_c row-major
  double mscale;
  double tol;
  int32_t max_iter;
  int32_t replay;        // 1 => active_j = iters_j < replay_iters[j]
  int32_t replay_iters[MAXC];
  int32_t ncol;
  int32_t mode;
  const double* lam0_src;  // lambda_0(theta) for the record: device scalar (times lam0_mul), or NULL => lam0_val
  double lam0_val;
  double lam0_mul;
  const int32_t* lz_info;  // {iterations, converged} of the Lanczos that produced lambda_0 (NULL: none)
};

// CG state for up to MAXC columns, updated only by "last CTA" finalisers.
struct CGState {
  double rr[MAXC];        // r^T r (current)
  double rr0[MAXC];       // ||rhs||^2
  double alpha[MAXC];
  double beta[MAXC];
  int32_t active[MAXC];
  int32_t iters[MAXC];
  int32_t any_active;
  int32_t par;            // ping-pong parity of the P / S(P) buffers
  int32_t hit_max;        // some column stopped at max_iter unconverged
  int32_t breakdown;      // some column met a non-finite r^T r or a non-finite / non-positive p^T q
  double quad;
  double t[MAXC];         // Pade trace terms
  unsigned int ticket[8]; // last-CTA counters (self-resetting)
};

enum FinKind { FIN_NONE = 0, FIN_INIT = 1, FIN_ALPHA = 2, FIN_UPDATE = 3, FIN_TRACE = 4 };
enum EpiKind { EPI_S = 0, EPI_DOT = 1 };

struct ApplyArgs {
  LayoutDev L;
  const EvalParams* prm;
  CGState* st;
  const double* u;         // [n_pad]
  const double* jitter;    // [n_c]
  // input D
  const double* D;         // [NC][n_pad]; with fuse_p this is R
  const double* S_D;       // [n_tiles][16] partials of S(D) (fuse_p: S(R))
  int fuse_p;              // D := R + beta o P_old (active columns), P_new written
  double* Pbuf[2];         // P ping-pong
  double* SPbuf[2];        // S(P) ping-pong partials
  int use_par_p2;          // P2 := Pbuf[par^1] (current search direction)
  // output
  double* out;
  const double* P2;        // combine term (or NULL)
  double cA[MAXC], cV[MAXC], cP[MAXC];
  int epi;                 // EpiKind
  double* Sout;            // EPI_S: partials of u^T out
  const double* Y2;        // EPI_DOT: partner of the dot
  double* dots;            // EPI_DOT: partials of out . Y2
  int fin;                 // FinKind (FIN_ALPHA or FIN_TRACE)
  int gate;                // return immediately when !st->any_active
  int ncol;
  double* alpha_hist;      // [MAXC][hist_stride]
  int hist_stride;
  int ld_max;
  int slot_doubles;        // TMA ring slot size (>= ld_max)
  int red_doubles;         // cross-k-group reduction scratch
  int nstage;              // TMA ring depth
  double* Tbuf;            // [n_c][MAXC] low-rank coefficients M' S (phase 1 of the apply)
  int nmine_max;           // max clusters per persistent CTA
  size_t smem_b, smem_nob; // dynamic shared memory with / without the ring
  int grid;                // persistent grid size
  int dbg;                 // timing experiments (NUGPR_APPLY_DBG); 0 in production
  int mma;                 // 3: DMMA column-task kernel, 2: staged DMMA, 1: DMMA, 0: DFMA
  int lds;                 // column-task kernel: padded column stride in shared memory
  int d_is_pnew;           // column-task kernel: D := P_new = Pbuf[par^1] (formed by pnew_kernel)
  int big;                 // big-block mode (ld_max > 512): row-tiled apply_big_kernel
  int f32;                 // 1: the DMMA apply streams the FP32-stored block (P->B32)
  int nw;                  // DMMA apply: consumer warps per CTA (7: 2 CTAs/SM; 3: 4 CTAs/SM)
  int dstride;             // DMMA apply: > 0 => D_i arrives per chunk with the TMA stream (stage row stride)
  int dbuf;                // DMMA apply: second D_i buffer; unfused applies prefetch the next cluster's D_i
};

struct ApplyPlan {
  int slot_doubles = 0, red_doubles = 0, nstage = 0, nmine_max = 0, grid = 0, ctas_per_sm = 0, mma = 0, lds = 0;
  int nw = 7;
  int dstride = 0;
  int dbuf = 0;
  size_t smem_b = 0, smem_nob = 0;
  bool ok = false;
};

struct LowrankArgs {
  const int32_t* task0;    // NULL: S partials per cluster; else per column task, cluster j = [task0[j], task0[j+1])
  const CGState* st;
  const EvalParams* prm;   // if set, M' is read from prm->Mp (mode-independent graphs)
  const double* Mp;        // n_c x n_c row-major (used when prm is NULL)
  const double* S;         // [n_tiles][16] S partials (tiles == clusters); fuse_p: S(R)
  double* SPbuf[2];        // fuse_p: S(P) ping-pong
  int fuse_p;
  double* T;               // [nrows][16] out: rows row0 .. row0+nrows-1 of M' S
  int n_c;                 // S / M' extent (all clusters, also when the clusters are sharded)
  int ncol;
  int gate;
  int row0, nrows;         // PAR-2: only this rank's clusters' rows of T (row0 = 0, nrows = n_c otherwise)
};

struct UpdateArgs {
  LayoutDev L;
  const EvalParams* prm;
  CGState* st;
  const double* u;
  double* X;
  double* R;
  const double* Q;
  double* Pbuf[2];
  double* rr_part;         // [n_tiles][16]
  double* SR_part;         // [n_tiles][16]
  double* beta_hist;       // [MAXC][hist_stride]
  int hist_stride;
  int ncol;
  unsigned long long cond; // cudaGraphConditionalHandle of the CG while-loop (0 = not in a graph)
  int nofin;               // PAR-2: no last-CTA finaliser (fin_kernel runs after the partials exchange)
};

struct RhsArgs {
  LayoutDev L;
  const EvalParams* prm;
  CGState* st;
  const double* Linv;
  const double* y;         // [n] cluster-sorted (unpadded)
  const double* probes;    // NULL or [m][n]
  uint64_t seed;
  const double* u;
  double* RHS;             // [NC][n_pad]
  double* R;
  double* X;
  double* P0;              // Pbuf[0]
  double* SP0;             // SPbuf[0]
  double* SR_part;
  double* rr_part;
  int ncol;
  const double* cy;        // NULL, or the precomputed transformed RHS c = R^{-T} y (padded layout)
  double* cy_out;          // NULL, or where to store c (first evaluation of a numgrad)
  int64_t pos0;            // PAR-2: global sorted position of this rank's first row (probe counter)
  int64_t n_glob;          // row count of the caller's probe matrix (= n when not sharded)
  int nofin;               // PAR-2: no last-CTA finaliser
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// splitmix64 counter generator (identical definition in synth/__init__.py `probes`).
__host__ __device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t ctr) {
  uint64_t x = seed + (ctr + 1ull) * 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ double probe_value(uint64_t seed, int j, int64_t p) {
  uint64_t ctr = (static_cast<uint64_t>(j) << 40) | static_cast<uint64_t>(p);
  return (splitmix64_at(seed, ctr) >> 63) ? -1.0 : 1.0;
}

// Kernel value.  Squared distance as sum_d (x_d - x'_d)^2 with explicitly non-fused ops
// (bitwise-symmetric blocks with an exact diagonal).
__device__ __forceinline__ double kval(int kind, double sq, double lam, double alpha) {
  if (kind == 0) {                       // RBF (reading X3)
    return alpha * exp(-__ddiv_rn(sq, 2.0 * lam * lam));
  } else if (kind == 2) {                // Eq. (2) as printed
    return alpha * exp(-__ddiv_rn(sqrt(sq), 2.0 * lam * lam));
  } else {                               // Matern-5/2
    double rho = sqrt(sq);
    double s = sqrt(5.0) * rho / lam;
    return alpha * (1.0 + s + 5.0 * sq / (3.0 * lam * lam)) * exp(-s);
  }
}

}  // namespace nugpr
