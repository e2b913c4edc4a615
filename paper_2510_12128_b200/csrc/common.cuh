// common.cuh — device-side layout and state shared by the nuGPR kernels.
//
// Internal data layout in HBM:
//  * Clusters are padded to ld_i = round_up(b_i, 8) rows ("padded rows", reading P19); the
//    padding rows are identity rows in every block matrix and zero in every vector, so they
//    are exactly invisible to the method.
//  * Vectors: column-major [NC][n_pad] FP64 (one contiguous length-n_pad column per RHS;
//    column 0 = the y-solve, columns 1..m = the Hutchinson probes).
//  * Block matrices: Linv_i dense ld_i x ld_i column-major at boff[i]; H_i and G_i (symmetric)
//    packed lower triangle in swizzled 8x8 tiles at pboff[i] (small layout, see swz below), or
//    full ld_i x ld_i at boff[i] in big-block mode (ld > 512).
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

// Packed symmetric block storage (small layout, ld <= 512; "only (K_diag, K_rep)
// need be stored", SURVEY §8(d) P = sum b(b+1)/2): only the lower triangle of H_i / G_i, in 8x8 tiles
// (I, K), I >= K (mt = ld/8 tiles per side), 64 elements per tile with element (r, c) at swz(r, c).
// Tiles are grouped in BLOCKS of up to 8x8 tiles: block (g, s) holds tiles I = 8g+a, K = 8s+b
// (a < h(g), b < h(s), h(x) = min(8, mt - 8x); a >= b when g == s), stored b-major; blocks are
// ordered column-block-major (s = 0.., then g = s..).  One block is one TMA chunk of the apply,
// and in it warp w does exactly the products of row a = w (out_I += T D_K) and column b = w
// (out_K += T^T D_I): regular, balanced work with no per-tile index search.  Diagonal tiles are
// stored full.  Within a tile, element (r, c) sits in 16-byte chunk pk_chunk(r, c/2) at half c&1:
// the DMMA splits k = 8 into k = 2 qc + h (h = 0, 1), so lane (qr, qc) reads its direct A pair
// T[qr][2qc..2qc+1] with one 16-byte load, and the chunk order (rows in pairs, columns XOR-rotated,
// parity-interleaved) makes both that load and the transposed loads T[2qc+h][qr] bank-conflict-free.
__host__ __device__ __forceinline__ int pk_chunk(int r, int j) {
  return 8 * (r >> 1) + ((j ^ ((r >> 1) & 3)) + 4 * ((r + j) & 1));
}
__host__ __device__ __forceinline__ int swz(int r, int c) { return 2 * pk_chunk(r, c >> 1) + (c & 1); }
__host__ __device__ __forceinline__ int64_t tri_tiles(int mt) { return static_cast<int64_t>(mt) * (mt + 1) / 2; }
__host__ __device__ __forceinline__ int pk_ns(int mt) { return (mt + 7) >> 3; }                 // block rows
__host__ __device__ __forceinline__ int pk_h(int x, int mt) { return (mt - 8 * x < 8) ? mt - 8 * x : 8; }
__host__ __device__ __forceinline__ int pk_nblocks(int mt) { const int ns = pk_ns(mt); return ns * (ns + 1) / 2; }
// first tile of block (g, s), g >= s: all column blocks before s are 8 tiles wide
__host__ __device__ __forceinline__ int pk_blk_off(int g, int s, int mt) {
  const int o = s * (8 * mt - 28) - 32 * s * (s - 1);
  if (g == s) return o;
  const int w = pk_h(s, mt);
  return o + w * (w + 1) / 2 + w * 8 * (g - s - 1);
}
__host__ __device__ __forceinline__ int pk_blk_size(int g, int s, int mt) {
  const int w = pk_h(s, mt);
  return (g == s) ? w * (w + 1) / 2 : pk_h(g, mt) * w;
}
// index of tile (I, K), I >= K, in the cluster's packed storage
__host__ __device__ __forceinline__ int pk_tile(int I, int K, int mt) {
  const int g = I >> 3, s = K >> 3, a = I & 7, b = K & 7;
  const int h = pk_h(g, mt);
  const int pos = (g == s) ? b * h - b * (b - 1) / 2 + (a - b) : b * h + a;
  return pk_blk_off(g, s, mt) + pos;
}

// One CTA's piece of the packed-block stream of an apply: blocks [k0, k1) (in storage order) of
// cluster blk.  The stream of all clusters is cut into PACK_CTAS pieces of equal tile count at block
// boundaries, so a cluster can be split over up to MAX_PARTS CTAs (part = its index); a split
// cluster's partial products meet in split scratch at `spoff` (doubles) and the last CTA to arrive
// (ticket `tick`) sums them in part order and runs the epilogue.
constexpr int PACK_CTAS = 148;   // B200 SM count: the partition is fixed (independent of the device)
constexpr int MAX_PARTS = 4;
struct SegDesc {
  int32_t blk, k0, k1, part, nparts, tick;
  int64_t spoff;
  int64_t t0;      // first tile of the piece in the packed buffer (a CTA's pieces are contiguous there)
  int32_t ntile;   // tiles in the piece
  int32_t pad_;
};

struct TileDesc {
  int32_t blk;    // cluster index
  int32_t row0;   // first padded row within the cluster
  int32_t nrows;  // rows in this tile (even)
  int32_t pad_;
};

struct LayoutDev {
  const int64_t* off;    // [n_c+1] original (unpadded) row offsets
  const int64_t* poff;   // [n_c+1] padded row offsets
  const int64_t* boff;   // [n_c] element offset of block i in full block storage (ld_i x ld_i)
  const int32_t* ld;     // [n_c] padded cluster size
  const TileDesc* tiles; // [n_tiles]
  const int32_t* tile0;  // [n_c+1] tile range of each cluster
  const int64_t* pboff;   // [n_c] element offset of block i in PACKED block storage (small layout)
  const SegDesc* segs;    // packed-apply pieces, CTA b owns segs[seg0[b] .. seg0[b+1])
  const int32_t* seg0;    // [n_seg_ctas + 1]
  int32_t n_c;
  int32_t n_tiles;
  int32_t n_seg_ctas;
  int32_t seg_max;        // max pieces per CTA
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
  const double* S_D;       // [lr_nc][MAXC] per-cluster S rows of D (fuse_p: S(R)); global under PAR-2
  int fuse_p;              // D := R + beta o P_old (active columns), P_new written
  double* Pbuf[2];         // P ping-pong
  double* SPbuf[2];        // S(P) ping-pong rows [lr_nc][MAXC]
  int use_par_p2;          // 1: P2 = Y2 := Pbuf[par^1]; 2: Y2 := D itself (mBCG)
  int lr_row0, lr_nc;      // low-rank term: M' rows of local cluster 0 (PAR-2 offset), S / M' extent
  // output
  double* out;
  const double* P2;        // combine term (or NULL)
  double cA[MAXC], cV[MAXC], cP[MAXC];
  int epi;                 // EpiKind
  double* Sout;            // EPI_S: per-cluster rows of u^T out
  const double* Y2;        // EPI_DOT: partner of the dot
  double* dots;            // EPI_DOT: per-cluster rows of out . Y2
  int fin;                 // FinKind (FIN_ALPHA or FIN_TRACE)
  int gate;                // return immediately when !st->any_active
  int ncol;
  double* alpha_hist;      // [MAXC][hist_stride]
  int hist_stride;
  // packed apply: split-cluster partial sums / tickets, launch plan
  double* split_part;
  unsigned int* split_ticket;
  int grid, slot_tiles, nstage, mtmax, nt8, f32, nacc, mst;
  int lr_stage_s;          // stage the S rows of the low-rank term in the ring (set by plan_packed_apply)
  size_t smem;
  int ld_max;
  // big-block path (ld > 512, apply_big_kernel): low-rank rows T = M'S from lowrank_kernel
  int big;
  double* Tbuf;            // [n_c][MAXC]
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
  double* SPbuf[2];        // S(P) rows ping-pong [n_c][MAXC]: the finaliser forms S(P_{k+1}) (cg_fin.cuh)
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
