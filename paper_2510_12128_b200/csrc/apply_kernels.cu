// apply_kernels.cu — row A3 of SURVEY §8(a): the fused multi-RHS apply of
// A = R^{-T} K''(theta) R^{-1} (Eq. 18-21, 23-25) on the PACKED symmetric blocks.
//
//   out = cA o (a D + b_i B_i D + u_i (mscale M' S(D))_i) + cV o D + cP o P2      per cluster i
//
// with B_i = H_i (noise / scale steps) or G_i(lambda') (lengthscale steps), the Q(A) / Pade-trace
// combines of PAPER.md:124 folded into (cA, cV, cP), and an epilogue that emits the next global
// reduction's per-cluster rows (S(out) = u_i^T out_i, or out . Y2 for the CG / trace dots).
//
// Design (B200):
//  * Only the lower triangle of each symmetric B_i is streamed (the packed
//    P = sum b(b+1)/2 of SURVEY §8(d)): 8x8 tiles in column-major tile order, each tile used for
//    both products it stands for — out_I += T D_K ("direct") and out_K += T^T D_I ("transposed") —
//    on the FP64 tensor pipe (mma.sync m8n8k4 f64: 8 probe columns per n8 tile), the y column as a
//    DFMA on the same A fragment.  Consumer warp w owns the output m-tiles w, w+8, ...
//  * One persistent CTA per SM: 8 consumer warps + 1 TMA producer warp.  The producer streams the
//    CTA's piece of the packed stream through an nstage-deep ring of 1-D bulk copies (full/empty
//    mbarriers) and stages each cluster's D inputs (and P_old for the fused first apply) with
//    bulk copies ahead of use.
//  * Load balance: the packed stream of ALL clusters is cut into PACK_CTAS pieces of equal tile
//    count at tile-column boundaries (host, make_layout), so every SM streams the same bytes; a
//    cluster cut between CTAs leaves partial products in split scratch and the last CTA to finish
//    (ticket) sums them in part order — deterministic — and runs the epilogue.
//  * The low-rank coefficients T_i = M'[i,:] S(D) (Eq. 19-21) are formed by the consumer warps at
//    kernel start from the previous kernel's per-cluster S rows, while the producer fills the ring:
//    no separate low-rank launch (for the fused first apply the update finaliser has formed the rows
//    S(P_new) = S(R) + beta S(P_old) already).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "cg_fin.cuh"
#include "common.cuh"
#include "kernels_decl.h"
#include "tma.cuh"

namespace nugpr {

#ifdef NUGPR_TRACE_APPLY
// diagnostics build only (build.py --trace): globaltimer stamps of one launch, per CTA
constexpr int TRACE_W = 64;
__device__ unsigned long long g_apply_trace[PACK_CTAS][TRACE_W];
__device__ int g_apply_trace_on;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TR(idx) do { if (g_apply_trace_on && (idx) < TRACE_W) g_apply_trace[blockIdx.x][(idx)] = gtimer(); } while (0)
#define TRV(idx, v) do { if (g_apply_trace_on) g_apply_trace[blockIdx.x][(idx)] = (v); } while (0)
#define TCLK(v) (v) = clock64()
#define TACC(idx, v) do { tacc_[(idx) - 48] += (v); } while (0)
#define TACC_DECL long long tacc_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define TACC_FLUSH do { if (g_apply_trace_on && wid == 0 && lane == 0) for (int i_ = 0; i_ < 8; ++i_) g_apply_trace[blockIdx.x][48 + i_] = tacc_[i_]; \
  if (g_apply_trace_on && lane == 0 && wid < 8) g_apply_trace[blockIdx.x][56 + wid] = tacc_[1] + tacc_[0]; } while (0)
#else
#define TCLK(v) do {} while (0)
#define TACC(idx, v) do {} while (0)
#define TACC_DECL
#define TACC_FLUSH do {} while (0)
#define TR(idx) do {} while (0)
#define TRV(idx, v) do {} while (0)
#endif

// NM MMA warps (8), warp w owning the output m-tiles w, w+NM, ...; a block's tile rows / columns
// w + NM rr (rr < 8 / NM)
constexpr int PNE_MAX = 7;             // epilogue warps
constexpr int LRG = 4;                 // pieces per pass of the low-rank rows (LRG x 4 accumulators per thread)
constexpr int CHUNK = 64;              // tiles per ring chunk (32 KB FP64)

// (not volatile: a pure function of its operands, so the compiler may schedule it freely)
__device__ __forceinline__ void dmma_pk(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int PNE>
__device__ __forceinline__ void bar_epi() { asm volatile("bar.sync 2, %0;" ::"r"(PNE * 32) : "memory"); }

template <typename TB>
__device__ __forceinline__ double ldA(const TB* p) { return static_cast<double>(*p); }
__device__ __forceinline__ double2 ldA2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ double2 ldA2(const float* p) {
  const float2 v = *reinterpret_cast<const float2*>(p);
  return make_double2(v.x, v.y);
}

// D buffer: column-major [NCP columns][ldp], column 0 = y; ldp = 8 (mod 16) doubles so that the
// 16-byte B-pair loads D[8t + 2qc + h][col qr] of a quarter warp (rows qr = 2t', 2t'+1) hit all banks
__host__ __device__ __forceinline__ int pk_ldp(int ld_max) { return ((ld_max + 15) & ~15) + 8; }
// rows of one Acc buffer: whole 8 x 8-tile block rows, so a cluster whose last block row is one tile
// high ("thin") can keep the other warps' partial products of that row in the tile rows past ld
__host__ __device__ __forceinline__ int pk_acc_rows(int ld_max) { return ((ld_max / 8 + 7) / 8) * 64; }

// Shared-memory plan (host and device agree): ring | Dp[2] | Acc[nacc] | Tsm (T rows of every piece,
// then the per-warp partials of one pass) | Mst (the M' rows of the CTA's pieces, when staged)
struct PackSmem {
  size_t ring, dp, acc, tsm, mst, total;
};
__host__ __device__ inline PackSmem pack_smem(int nstage, int esize, int ld_max, int nt8, int pne, int seg_max,
                                              int nacc, int64_t mst_doubles) {
  PackSmem p;
  const size_t ncp = 1 + 8 * static_cast<size_t>(nt8);
  p.ring = 0;
  size_t o = static_cast<size_t>(nstage) * CHUNK * 64 * esize;
  o = (o + 127) / 128 * 128;
  p.dp = o;
  o += 2 * ncp * pk_ldp(ld_max) * sizeof(double);
  p.acc = o;                                      // nacc x block products [ld_max][NCP]
  o += static_cast<size_t>(nacc) * pk_acc_rows(ld_max) * ncp * sizeof(double);
  p.tsm = o;
  o += static_cast<size_t>(seg_max + pne * LRG) * MAXC * sizeof(double);
  o = (o + 127) / 128 * 128;
  p.mst = o;
  o += static_cast<size_t>(mst_doubles) * sizeof(double);
  p.total = o;
  return p;
}


// Warp-specialised persistent apply: 8 MMA warps stream the CTA's tile blocks, the epilogue warps form
// the next piece's D, the low-rank rows and the previous piece's epilogue (and the split-cluster
// combine, the finaliser), 1 warp drives the TMA ring.  Handshakes (mbarriers):
//   full / empty [nstage]      producer <-> MMA warps (one 64-tile chunk of the stream per slot)
//   dready[2]                  epilogue -> MMA (D of piece q formed in Dp[q&1])
//   accready / accfree [2]     MMA -> epilogue (block products of piece q in Acc[q % nacc]; Dp[q&1]
//                              is free again) / epilogue -> MMA (Acc[x] consumed).  With nacc = 2
//                              the MMA warps run a piece ahead of the epilogue (whose first piece
//                              waits for the low-rank rows)
template <int NM, int MTMAX, int NT8, typename TB, int PNE>
__global__ void __launch_bounds__((NM + PNE + 1) * 32, 8 / NM) apply_packed_kernel(const __grid_constant__ ApplyArgs a) {
  constexpr int PNM = NM, PWE = NM;              // MMA warps; the first epilogue warp
  constexpr int RR = 8 / NM;                     // tile rows / columns per MMA warp in a block
  constexpr int NCP = 1 + 8 * NT8;               // y + probe columns held per row
  constexpr int PWP = PNM + PNE;                 // the TMA producer warp
  if (a.gate && !a.st->any_active) return;
  const int b = blockIdx.x;
  const int s_lo = a.L.seg0[b], s_hi = a.L.seg0[b + 1];
  const int nseg = s_hi - s_lo;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t empty[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t dready[2], dbar[2], accready[2], accfree[2], mfull;
  __shared__ double ered[PNE_MAX * MAXC];
  __shared__ double cb[2 * MAXC];
  __shared__ int s_last;
  const int nacc = a.nacc;
  const int64_t mst_doubles = a.mst ? static_cast<int64_t>(a.L.seg_max) * a.lr_nc : 0;
  const PackSmem L_ = pack_smem(a.nstage, static_cast<int>(sizeof(TB)), a.ld_max, NT8, PNE, a.L.seg_max, nacc, mst_doubles);
  TB* ring = reinterpret_cast<TB*>(smraw + L_.ring);
  double* Dpb = reinterpret_cast<double*>(smraw + L_.dp);   // [2][NCP][ldp]
  double* Accb = reinterpret_cast<double*>(smraw + L_.acc); // nacc x [ld_max][NCP] block products of a piece
  const int accstride = pk_acc_rows(a.ld_max) * NCP;
  double* Tsm = reinterpret_cast<double*>(smraw + L_.tsm);  // T rows [seg_max][MAXC], then partials
  double* Mst = reinterpret_cast<double*>(smraw + L_.mst);  // [seg][lr_nc] staged M' rows (a.mst)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n_pad = a.L.n_pad;
  const int ncol = a.ncol;
  const EvalParams* P = a.prm;
  const int par = a.st->par;
  const TB* B = (sizeof(TB) == 4) ? reinterpret_cast<const TB*>(P->B32) : reinterpret_cast<const TB*>(P->B);
  const bool useB = (P->B != nullptr);
  const int nstage = a.nstage;
  const int ldp = pk_ldp(a.ld_max);
  const int dpstride = NCP * ldp;                            // one D buffer
  const double* Pold = a.fuse_p ? a.Pbuf[par] : nullptr;
  double* Pnew = a.fuse_p ? a.Pbuf[par ^ 1] : nullptr;
  // the low-rank coefficients' input rows S(D) ([lr_nc][MAXC], 128 B each) are staged by one bulk copy
  // into the first lrk ring slots when they fit while >= 2 slots stay for the block stream; those
  // slots join the stream once the low-rank rows of all pieces are formed (virtual chunks 0 .. lrk-1)
  const size_t slot_bytes = static_cast<size_t>(CHUNK) * 64 * sizeof(TB);
  const size_t s_bytes = static_cast<size_t>(a.lr_nc) * MAXC * sizeof(double);
  const int lrk_need = static_cast<int>((s_bytes + slot_bytes - 1) / slot_bytes);
  const int lrk = (a.lr_stage_s && a.lr_nc > 0 && lrk_need <= (useB ? nstage - 2 : nstage)) ? lrk_need : 0;
  const double* P2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.P2;
  const double* Y2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.Y2;
  long long clk_start = 0;
  TCLK(clk_start);
  if (tid == 0) {
    TR(0);
    TRV(46, nseg);
    for (int s_ = 0; s_ < nstage; ++s_) { mbar_init(&full[s_], 1); mbar_init(&empty[s_], PNM); }
    for (int k = 0; k < 2; ++k) { mbar_init(&dready[k], 1); mbar_init(&dbar[k], 1); }
    for (int k = 0; k < 2; ++k) { mbar_init(&accready[k], PNM); mbar_init(&accfree[k], 1); }
    mbar_init(&mfull, 1);
    fence_mbar_init();
  }
  if (tid < MAXC) {
    cb[tid] = (tid < ncol) ? a.st->beta[tid] : 0.0;
    cb[MAXC + tid] = (tid < ncol) ? static_cast<double>(a.st->active[tid]) : 0.0;
  }
  __syncthreads();

  // registers: the two MMA warpgroups take 168 per thread, the epilogue / producer warpgroup 88
  // (entry: 128 x 16 warps = the whole register file); the MMA block loop needs the headroom to issue
  // its shared-memory operand loads ahead of the DMMAs
  static_assert(NM == 8 && PNE == 7, "setmaxnreg split assumes warpgroups {MMA, MMA, epilogue+producer}");
  if (wid < PNM) asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n" ::: "memory");
  else asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");

  if (wid == PWP) {
    // ================================ TMA producer ================================
    if (lane == 0 && nseg > 0) {
      if (a.mst) {
        // the M' rows of this CTA's pieces first (HBM reads at the head of the queue)
        const uint32_t rb = static_cast<uint32_t>(a.lr_nc) * 8u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&mfull, rb * static_cast<uint32_t>(nseg));
        for (int q = 0; q < nseg; ++q)
          tma_load_1d(Mst + static_cast<int64_t>(q) * a.lr_nc,
                      P->Mp + static_cast<int64_t>(a.lr_row0 + a.L.segs[s_lo + q].blk) * a.lr_nc, rb, &mfull);
      }
      if (lrk > 0) {
        const double* SDp = a.fuse_p ? a.SPbuf[par] : a.S_D;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[0], static_cast<uint32_t>(s_bytes));
        tma_load_1d(ring, SDp, static_cast<uint32_t>(s_bytes), &full[0]);
        for (int k = 1; k < lrk; ++k) mbar_arrive(&full[k]);
      }
      // (not staged) the M' rows of this CTA's pieces into L2 (the epilogue warps' low-rank rows read
      // them early; behind the block stream they would wait in the DRAM queues)
      if (!a.mst && (a.lr_nc & 1) == 0)             // (bulk prefetch: 16-byte aligned rows)
        for (int q = 0; q < nseg; ++q)
          tma_prefetch_l2(P->Mp + static_cast<int64_t>(a.lr_row0 + a.L.segs[s_lo + q].blk) * a.lr_nc,
                          static_cast<uint32_t>(a.lr_nc) * 8u);
      if (useB) {
        // the CTA's stream: tiles [t0, t0 + ntot) of the packed buffer, in CHUNK-tile copies
        const int64_t t0 = a.L.segs[s_lo].t0;
        const SegDesc last = a.L.segs[s_hi - 1];
        const int64_t ntot = last.t0 + last.ntile - t0;
        const int nchunk = static_cast<int>((ntot + CHUNK - 1) / CHUNK);
        // warm L2 with the epilogue inputs of every piece (plain loads in the epilogue)
        for (int q = 0; q < nseg; ++q) {
          const int i = a.L.segs[s_lo + q].blk;
          const int64_t p0 = a.L.poff[i];
          const uint32_t cbytes = static_cast<uint32_t>(a.L.ld[i]) * 8u;
          tma_prefetch_l2(a.u + p0, cbytes);
          for (int c = 0; c < ncol; ++c) {
            if (P2) tma_prefetch_l2(P2 + c * n_pad + p0, cbytes);
            if (a.epi == EPI_DOT && Y2 && Y2 != P2) tma_prefetch_l2(Y2 + c * n_pad + p0, cbytes);
          }
        }
        // chunks = runs of consecutive blocks of <= CHUNK tiles (a block never straddles two chunks, so
        // the MMA warps address a block's tiles at constant offsets from its base)
        int s_ = lrk, c = lrk;                       // (virtual chunks 0 .. lrk-1: the S staging)
        uint32_t ph = 0;
        int64_t cstart = t0;
        int cfill = 0;
        auto issue = [&]() {
          if (c >= nstage) mbar_wait_sleep(&empty[s_], ph ^ 1u, 64);
          const uint32_t bytes = static_cast<uint32_t>(cfill) * 64u * static_cast<uint32_t>(sizeof(TB));
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full[s_], bytes);
          tma_load_1d(ring + static_cast<int64_t>(s_) * CHUNK * 64, B + cstart * 64, bytes, &full[s_]);
          if (++s_ == nstage) { s_ = 0; ph ^= 1u; }
          ++c;
          cstart += cfill;
          cfill = 0;
        };
        for (int q = 0; q < nseg; ++q) {
          const SegDesc sd = a.L.segs[s_lo + q];
          const int mt = a.L.ld[sd.blk] >> 3, ns = pk_ns(mt);
          int sb = 0, gb = 0;
          for (int k = 0; k < sd.k0; ++k) { if (++gb == ns) { ++sb; gb = sb; } }
          for (int k = sd.k0; k < sd.k1; ++k) {
            const int nt = pk_blk_size(gb, sb, mt);
            if (cfill + nt > CHUNK) issue();
            cfill += nt;
            if (++gb == ns) { ++sb; gb = sb; }
          }
        }
        if (cfill > 0) issue();
        (void)ntot;
        (void)nchunk;
      }
      TR(2);
    }
    return;
  }


  if (wid < PNM) {
    // ================================ MMA warps ================================
    if (!useB) return;                               // no block term: the epilogue warps do everything
    const int qr = lane >> 2, qc = lane & 3;
    // k = 2 qc + h: direct A pair T[qr][2qc + h] (one 16-byte load), transposed A T[2qc + h][qr]
    const int offD = swz(qr, 2 * qc), offT0 = swz(2 * qc, qr), offT1 = swz(2 * qc + 1, qr);
    const int bo = (1 + qr) * ldp + 2 * qc;          // B pair D[8t + 2qc + h][probe qr] at bo + 8t
    // chunk bookkeeping (the producer's walk): the current chunk sits in slot cs, filled up to cfill tiles
    int ws = lrk, cs = -1;
    uint32_t wph = 0;
    int cfill = CHUNK;
    TACC_DECL
    for (int q = 0; q < nseg; ++q) {
      const SegDesc sd = a.L.segs[s_lo + q];
      const int mt = a.L.ld[sd.blk] >> 3;
      const double* Dp = Dpb + (q & 1) * dpstride;
      long long tp0 = 0, tp1 = 0, tp2 = 0, tp3 = 0, tp4 = 0;
      TCLK(tp0);
      mbar_wait_sleep(&dready[q & 1], static_cast<uint32_t>((q >> 1) & 1), 128);
      TCLK(tp1);
      if (lane == 0) TACC(50, tp1 - tp0);
      if (wid == 0 && lane == 0 && q < 8) TR(4 + q);
      double acc[NT8][2][MTMAX], accy[MTMAX];
#pragma unroll
      for (int j = 0; j < MTMAX; ++j) {
        accy[j] = 0.0;
#pragma unroll
        for (int n = 0; n < NT8; ++n) { acc[n][0][j] = 0.0; acc[n][1][j] = 0.0; }
      }
      const int ns = pk_ns(mt);
      // thin last block row (one tile high): its direct products go to the warp owning the tile
      // COLUMN (warp b: tile (last, 8s + b)), each into its unused accumulator slot of that block row;
      // the epilogue sums the eight partial rows in warp order
      const bool thin = NM == 8 && ns > 1 && pk_h(ns - 1, mt) == 1;
      int sb = 0, gb = 0;
      for (int k = 0; k < sd.k0; ++k) { if (++gb == ns) { ++sb; gb = sb; } }
      for (int k = sd.k0; k < sd.k1; ++k) {
        const int h = pk_h(gb, mt), w = pk_h(sb, mt);
        const bool diag = gb == sb;
        const int nt = diag ? w * (w + 1) / 2 : h * w;
        long long tw0 = 0, tw1 = 0;
        TCLK(tw0);
        if (cfill + nt > CHUNK) {                    // next chunk: hand back the current one, wait for it
          if (cs >= 0) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[cs]);
          }
          cs = ws;
          mbar_wait_sleep(&full[ws], wph, 32);
          if (++ws == nstage) { ws = 0; wph ^= 1u; }
          cfill = 0;
        }
        TCLK(tw1);
        if (lane == 0) TACC(48, tw1 - tw0);
        const TB* blk = ring + (static_cast<int64_t>(cs) * CHUNK + cfill) * 64;
        auto tile = [&](int pos) -> const TB* { return blk + pos * 64; };
        // one k-tile step: x[hh] += A_hh D[k-tile kt] (hh = 0, 1 independent DMMA chains), and the y column
        auto step = [&](double (&x0)[2][NT8], double (&x1)[2][NT8], double& xy, double a0, double a1, int kt) {
          const double* db = Dp + bo + kt * 8;
#pragma unroll
          for (int n = 0; n < NT8; ++n) {
            const double2 bv = *reinterpret_cast<const double2*>(db + n * 8 * ldp);
            dmma_pk(x0[0][n], x1[0][n], a0, bv.x);
            dmma_pk(x0[1][n], x1[1][n], a1, bv.y);
          }
          const double2 yv = *reinterpret_cast<const double2*>(Dp + kt * 8 + 2 * qc);
          xy = fma(a1, yv.y, fma(a0, yv.x, xy));
        };
        auto fold = [&](double (&x0)[2][NT8], double (&x1)[2][NT8], double& xy, int jt) {
#pragma unroll
          for (int j = 0; j < MTMAX; ++j)
            if (j == jt) {
#pragma unroll
              for (int n = 0; n < NT8; ++n) {
                acc[n][0][j] += x0[0][n] + x0[1][n];
                acc[n][1][j] += x1[0][n] + x1[1][n];
              }
              accy[j] += xy;
            }
        };
        auto zero = [&](double (&x0)[2][NT8], double (&x1)[2][NT8], double& xy) {
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int n = 0; n < NT8; ++n) { x0[e][n] = 0.0; x1[e][n] = 0.0; }
          xy = 0.0;
        };
        // warp wid does the tile rows / columns wa = wid + NM rr of the block (rr < 8 / NM)
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
          const int wa = wid + NM * rr;
          double d0[2][NT8], d1[2][NT8], dy, t0[2][NT8], t1[2][NT8], ty;
          zero(d0, d1, dy);
          zero(t0, t1, ty);
          if (h == 8 && w == 8) {
            if (diag) {
              // diagonal block: row wa of the lower triangle, the tiles (wa, kk) kk <= wa direct and
              // (kk, wa) kk > wa transposed — both give rows 8g + wa from D rows 8kk (branch-free).
              // All A operands are loaded first (shared-memory latency overlaps the DMMA chains).
              double A0[8], A1[8];
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const bool dir = kk <= wa;
                const int pos = dir ? 8 * kk - kk * (kk - 1) / 2 + (wa - kk) : 8 * wa - wa * (wa - 1) / 2 + (kk - wa);
                const TB* tp = tile(pos);
                A0[kk] = ldA(tp + (dir ? offD : offT0));
                A1[kk] = ldA(tp + (dir ? offD + 1 : offT1));
              }
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) step(d0, d1, dy, A0[kk], A1[kk], 8 * sb + kk);
              fold(d0, d1, dy, gb * RR + rr);
            } else {
              // off-diagonal block: direct tile (wa, kk) -> rows 8g + wa, transposed (kk, wa) -> rows 8s + wa
              double2 AD[8];
              double AT0[8], AT1[8];
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                AD[kk] = ldA2(tile(8 * kk + wa) + offD);
                const TB* tpt = tile(8 * wa + kk);
                AT0[kk] = ldA(tpt + offT0);
                AT1[kk] = ldA(tpt + offT1);
              }
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                step(d0, d1, dy, AD[kk].x, AD[kk].y, 8 * sb + kk);
                step(t0, t1, ty, AT0[kk], AT1[kk], 8 * gb + kk);
              }
              fold(d0, d1, dy, gb * RR + rr);
              fold(t0, t1, ty, sb * RR + rr);
            }
          } else {
            // edge block (the last block row / column of a cluster whose ld is not a multiple of 64)
            if (wa < w) {                                     // transposed: column b = wa
              const int bcol = wa;
              const int cbase = diag ? bcol * h - bcol * (bcol - 1) / 2 - bcol : bcol * h;   // tile (a, b) at cbase + a
              for (int aa = diag ? bcol + 1 : 0; aa < h; ++aa) {
                const TB* tp = tile(cbase + aa);
                step(t0, t1, ty, ldA(tp + offT0), ldA(tp + offT1), 8 * gb + aa);
              }
              fold(t0, t1, ty, sb * RR + rr);
            }
            if (thin && h == 1 && !diag) {                    // thin row, split by tile column
              if (wa < w) {
                const double2 ad = ldA2(tile(wa) + offD);
                step(d0, d1, dy, ad.x, ad.y, 8 * sb + wa);
                fold(d0, d1, dy, gb * RR + rr);
              }
            } else if (wa < h) {                              // direct: row a = wa
              const int arow = wa;
              const int b_hi = diag ? arow : w - 1;
              for (int bb = 0; bb <= b_hi; ++bb) {
                const int pos = diag ? bb * h - bb * (bb - 1) / 2 + (arow - bb) : bb * h + arow;
                const double2 ad = ldA2(tile(pos) + offD);
                step(d0, d1, dy, ad.x, ad.y, 8 * sb + bb);
              }
              fold(d0, d1, dy, gb * RR + rr);
            }
          }
        }
        long long tw2 = 0;
        TCLK(tw2);
        if (lane == 0) {
          TACC(49, tw2 - tw1);
        }
        cfill += nt;
        if (++gb == ns) { ++sb; gb = sb; }
      }
      TCLK(tp2);
      // y column: sum the 4 k-lanes of each row quad
#pragma unroll
      for (int j = 0; j < MTMAX; ++j) {
        accy[j] += __shfl_xor_sync(0xffffffffu, accy[j], 1);
        accy[j] += __shfl_xor_sync(0xffffffffu, accy[j], 2);
      }
      TCLK(tp3);
      if (lane == 0) { TACC(52, tp3 - tp2); TACC(53, tp3 - tp1); }
      if (wid == 0 && lane == 0 && q < 8) TR(12 + q);
      const int ax = q % nacc;
      mbar_wait_sleep(&accfree[ax], static_cast<uint32_t>((q / nacc) & 1), 128);
      double* Acc = Accb + ax * accstride;
      TCLK(tp4);
      if (lane == 0) TACC(51, tp4 - tp3);
      if (wid == 0 && lane == 0 && q < 8) TR(20 + q);
#pragma unroll
      for (int j = 0; j < MTMAX; ++j) {
        const int mtj = wid + j * PNM;
        if (mtj < mt || (thin && mtj < 8 * ns)) {
          double* row = Acc + (8 * mtj + qr) * NCP;
          if (qc == 0) row[0] = accy[j];
#pragma unroll
          for (int n = 0; n < NT8; ++n) {
            row[1 + 8 * n + 2 * qc] = acc[n][0][j];
            row[2 + 8 * n + 2 * qc] = acc[n][1][j];
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&accready[ax]);
    }
    TACC_FLUSH;
    return;
  }

  // ================================ epilogue warps ================================
  const int et = tid - PWE * 32;                     // 0 .. 32 PNE - 1
  const int ew = wid - PWE;
  const int NET = PNE * 32;
  // the low-rank coefficients' input rows: S(D) of the previous kernel, or for the fused apply the
  // S(P_new) rows the update finaliser formed (cg_fin.cuh)
  const double* SD = a.fuse_p ? a.SPbuf[par] : a.S_D;
  // D of piece q into Dp[q&1] by bulk copies, one per column (fused: R into Dp, P_old staged in
  // Acc[q % nacc]); issued by one thread, completing on dbar[q&1]
  auto issue_d = [&](int q) {
    double* Acc = Accb + (q % nacc) * accstride;
    const SegDesc sd = a.L.segs[s_lo + q];
    const int ld = a.L.ld[sd.blk];
    const int64_t p0 = a.L.poff[sd.blk];
    double* Dp = Dpb + (q & 1) * dpstride;
    const uint32_t bytes = static_cast<uint32_t>(ld) * 8u;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&dbar[q & 1], bytes * static_cast<uint32_t>(ncol) * (a.fuse_p ? 2u : 1u));
    for (int c = 0; c < ncol; ++c) {
      tma_load_1d(Dp + c * ldp, a.D + c * n_pad + p0, bytes, &dbar[q & 1]);
      if (a.fuse_p) tma_load_1d(Acc + c * ld, Pold + c * n_pad + p0, bytes, &dbar[q & 1]);
    }
  };
  // fused apply: D = R + beta o P_old (active columns), P_old for inactive ones; P_new written by part 0
  auto fuse_d = [&](int q) {
    const double* Acc = Accb + (q % nacc) * accstride;
    const SegDesc sd = a.L.segs[s_lo + q];
    const int ld = a.L.ld[sd.blk];
    const int64_t p0 = a.L.poff[sd.blk];
    double* Dp = Dpb + (q & 1) * dpstride;
    for (int idx = et; idx < ld * ncol; idx += NET) {
      const int c = idx / ld, k = idx - c * ld;
      const double po = Acc[c * ld + k];
      const double x = (cb[MAXC + c] != 0.0) ? Dp[c * ldp + k] + cb[c] * po : po;
      Dp[c * ldp + k] = x;
      if (sd.part == 0) Pnew[c * n_pad + p0 + k] = x;
    }
  };
  // form D of piece q in Dp[q&1] with plain loads (the apply without a block term)
  auto form_d = [&](int q) {
    const SegDesc sd = a.L.segs[s_lo + q];
    const int ld = a.L.ld[sd.blk];
    const int64_t p0 = a.L.poff[sd.blk];
    double* Dp = Dpb + (q & 1) * dpstride;
    for (int idx = et; idx < ld * ncol; idx += NET) {
      const int c = idx / ld, k = idx - c * ld;
      const int64_t gi = c * n_pad + p0 + k;
      double x = __ldg(a.D + gi);
      if (a.fuse_p) {
        const double po = __ldg(Pold + gi);
        x = (cb[MAXC + c] != 0.0) ? x + cb[c] * po : po;
        if (sd.part == 0) Pnew[gi] = x;
      }
      Dp[c * ldp + k] = x;
    }
  };
  // the D of piece q has landed (fused: combine it); then signal the MMA warps (and release
  // Acc[q % nacc], which staged P_old: it is next written by the MMA warps' piece q - 2 + nacc)
  auto finish_d = [&](int q, bool rel) {
    mbar_wait_sleep(&dbar[q & 1], static_cast<uint32_t>((q >> 1) & 1), 64);
    if (a.fuse_p) {
      fuse_d(q);
      bar_epi<PNE>();
    }
    if (et == 0) {
      if (rel) mbar_arrive(&accfree[q % nacc]);
      mbar_arrive(&dready[q & 1]);
    }
  };
  if (useB) {
    // prologue: D of the first two pieces (fused with one Acc: one at a time, P_old staged in it)
    if (et == 0) {
      issue_d(0);
      if ((!a.fuse_p || nacc == 2) && nseg > 1) issue_d(1);
    }
    if (a.fuse_p) {
      finish_d(0, nseg == 1 || nacc == 2);
      if (nseg > 1) {
        if (et == 0 && nacc == 1) issue_d(1);
        finish_d(1, true);
      }
    } else {
      if (et == 0)                                   // Acc was never a staging buffer
        for (int x = 0; x < nacc; ++x) mbar_arrive(&accfree[x]);
      finish_d(0, false);
      if (nseg > 1) finish_d(1, false);
    }
  }
  double* Tpart = Tsm + a.L.seg_max * MAXC;          // [PNE][LRG][MAXC] per-warp partials
  // low-rank rows T_q = M'[row(q), :] S(D) of pieces [q0, q0 + LRG) into Tsm[q].  Thread et owns
  // columns 4 cg .. 4 cg + 3 (cg = et % 4) of the S rows j = et / 4 + (NET / 4) k; each (piece, column)
  // sum runs over j in that fixed order, then over the 8 row lanes of a warp (butterfly) and the warps in
  // order: the same bits on every CTA, for any set of pieces, whatever the partition.
  auto lr_rows = [&](int q0) {
    const int nc = a.lr_nc;
    const int cg = et & 3, jl = et >> 2, NJ = NET / 4;
    const int nq = min(LRG, nseg - q0);
    const bool cact = 4 * cg < ncol;
    const double* Mr[LRG];
#pragma unroll
    for (int g = 0; g < LRG; ++g)
      Mr[g] = a.mst ? Mst + static_cast<int64_t>(q0 + min(g, nq - 1)) * nc
                    : P->Mp + static_cast<int64_t>(a.lr_row0 + a.L.segs[s_lo + q0 + min(g, nq - 1)].blk) * nc;
    double t[LRG][4];
#pragma unroll
    for (int g = 0; g < LRG; ++g)
#pragma unroll
      for (int u = 0; u < 4; ++u) t[g][u] = 0.0;
    if (cact) {
      const double* Sst = reinterpret_cast<const double*>(smraw + L_.ring);
#pragma unroll 4
      for (int j = jl; j < nc; j += NJ) {
        double2 s01, s23;
        if (lrk > 0) {
          const double2* sr = reinterpret_cast<const double2*>(Sst + j * MAXC + 4 * cg);
          s01 = sr[0];
          s23 = sr[1];
        } else {
          const double2* sr = reinterpret_cast<const double2*>(SD + static_cast<int64_t>(j) * MAXC + 4 * cg);
          s01 = __ldcg(sr);
          s23 = __ldcg(sr + 1);
        }
        const double x[4] = {s01.x, s01.y, s23.x, s23.y};
        double m[LRG];
#pragma unroll
        for (int g = 0; g < LRG; ++g) m[g] = a.mst ? Mr[g][j] : __ldg(Mr[g] + j);
#pragma unroll
        for (int g = 0; g < LRG; ++g)
#pragma unroll
          for (int u = 0; u < 4; ++u) t[g][u] = fma(m[g], x[u], t[g][u]);
      }
    }
    // the 8 row lanes of the warp (lane = 4 jl' + cg), butterfly in fixed order
#pragma unroll
    for (int g = 0; g < LRG; ++g)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double v = t[g][u];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        t[g][u] = v;
      }
    if (lane < 4)
#pragma unroll
      for (int g = 0; g < LRG; ++g)
#pragma unroll
        for (int u = 0; u < 4; ++u) Tpart[(ew * LRG + g) * MAXC + 4 * lane + u] = t[g][u];
    bar_epi<PNE>();
    if (et < nq * MAXC) {
      const int g = et >> 4, cc = et & 15;
      double acc_ = 0.0;
      for (int w = 0; w < PNE; ++w) acc_ += Tpart[(w * LRG + g) * MAXC + cc];
      Tsm[(q0 + g) * MAXC + cc] = acc_;
    }
    bar_epi<PNE>();
  };
  int pend = -1;                                     // a piece whose D copy is in flight
  for (int q = 0; q < nseg; ++q) {
    const SegDesc sd = a.L.segs[s_lo + q];
    const int i = sd.blk, ld = a.L.ld[i];
    const int64_t p0 = a.L.poff[i];
    const double* Dp = Dpb + (q & 1) * dpstride;      // D of this piece (kept until its epilogue)
    double* Acc = Accb + (q % nacc) * accstride;      // its block products
    if (!useB) {
      form_d(q);                                     // (no block term: the epilogue warps form D here)
      bar_epi<PNE>();
    }
    if (pend >= 0) { finish_d(pend, a.fuse_p); pend = -1; }
    if (a.mst && q == 0) {
      mbar_wait_sleep(&mfull, 0u, 64);
      if (et == 0) TR(1);
    }
    if (lrk > 0) {
      if (q == 0) {
        // staged S: the low-rank rows of every piece now, then the staging slots go to the stream
        mbar_wait_sleep(&full[0], 0u, 64);
        if (et == 0) TR(3);
        for (int q0 = 0; q0 < nseg; q0 += LRG) lr_rows(q0);
        if (et == 0)
          for (int k = 0; k < lrk; ++k) mbar_arrive_cnt(&empty[k], PNM);
      }
    } else if (q % LRG == 0) {
      lr_rows(q);                                    // low-rank rows of pieces q .. q + LRG - 1
    }
    if (et == 0 && q == 0) TR(28);
    // register prefetch of this piece's epilogue inputs for the first row of every thread (the
    // latency hides behind the wait for the MMA warps)
    const bool pf = et < ld;
    double pf_u = 0.0, pf_p2[NCP], pf_y2[NCP];
    if (pf) {
      pf_u = __ldg(a.u + p0 + et);
#pragma unroll
      for (int c = 0; c < NCP; ++c) {
        const int64_t gi = c * n_pad + p0 + et;
        const bool on = c < ncol;
        pf_p2[c] = (on && P2) ? P2[gi] : 0.0;
        pf_y2[c] = (on && a.epi == EPI_DOT && a.use_par_p2 == 0) ? Y2[gi] : 0.0;
      }
    }
    bool run_epi = true;
    if (useB) {
      mbar_wait_sleep(&accready[q % nacc], static_cast<uint32_t>((q / nacc) & 1), 256);
      if (et == 0 && q < 8) TR(29 + q);
      {
        // thin last block row: its rows' products are split over eight partial tile rows
        const int mtq = ld >> 3, nsq = pk_ns(mtq);
        if (nsq > 1 && pk_h(nsq - 1, mtq) == 1) {
          const int r0 = ld - 8;
          for (int idx = et; idx < 8 * NCP; idx += NET) {
            const int rr = idx / NCP, c = idx - rr * NCP;
            double v = Acc[(r0 + rr) * NCP + c];
#pragma unroll
            for (int bb = 1; bb < 8; ++bb) v += Acc[(r0 + 8 * bb + rr) * NCP + c];
            Acc[(r0 + rr) * NCP + c] = v;
          }
          bar_epi<PNE>();
        }
      }
      // split cluster: publish this part's block products; the last part sums all parts in order
      if (sd.nparts > 1) {
        double* base = a.split_part + sd.spoff + static_cast<int64_t>(sd.part) * ld * NCP;
        for (int idx = et; idx < ld * NCP; idx += NET) base[idx] = Acc[idx];
        __threadfence();
        bar_epi<PNE>();
        if (et == 0) s_last = (atomicAdd(&a.split_ticket[sd.tick], 1u) == static_cast<unsigned>(sd.nparts - 1));
        bar_epi<PNE>();
        run_epi = s_last != 0;
        if (run_epi) {
          __threadfence();
          const double* all = a.split_part + sd.spoff;
          const int64_t pst = static_cast<int64_t>(ld) * NCP;
          for (int base2 = et; base2 < ld * NCP; base2 += 2 * NET) {
            double v[2][MAX_PARTS];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int pp = 0; pp < MAX_PARTS; ++pp) {
                const int idx = base2 + u * NET;
                v[u][pp] = (idx < ld * NCP && pp < sd.nparts) ? __ldcg(all + pp * pst + idx) : 0.0;
              }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int idx = base2 + u * NET;
              if (idx < ld * NCP) {
                double acc_ = v[u][0];
                for (int pp = 1; pp < sd.nparts; ++pp) acc_ += v[u][pp];
                Acc[idx] = acc_;
              }
            }
          }
          if (et == 0) a.split_ticket[sd.tick] = 0u;
        }
      }
    } else if (sd.part != 0) {
      run_epi = false;                               // no block term: part 0 holds the whole result
    }
    bar_epi<PNE>();                                  // T row (and the combined Acc) visible
    // epilogue: thread et owns rows r = et, et + 32 PNE, ...; D from Dp (shared), the block products
    // from Acc, the other inputs from global (coalesced over r for every column c)
    double ep[NCP];
#pragma unroll
    for (int c = 0; c < NCP; ++c) ep[c] = 0.0;
    if (run_epi) {
      const double bi = P->b0 + P->b1 * a.jitter[i];
      const double pa = P->a, ms = P->mscale;
      for (int r = et; r < ld; r += NET) {
        double uu, p2v[NCP], y2v[NCP];
        if (r == et) {
          uu = pf_u;
#pragma unroll
          for (int c = 0; c < NCP; ++c) { p2v[c] = pf_p2[c]; y2v[c] = pf_y2[c]; }
        } else {
          uu = __ldg(a.u + p0 + r);
#pragma unroll
          for (int c = 0; c < NCP; ++c) {
            const int64_t gi = c * n_pad + p0 + r;
            const bool on = c < ncol;
            p2v[c] = (on && P2) ? P2[gi] : 0.0;
            y2v[c] = (on && a.epi == EPI_DOT && a.use_par_p2 == 0) ? Y2[gi] : 0.0;
          }
        }
#pragma unroll
        for (int c = 0; c < NCP; ++c) {
          if (c >= ncol) continue;
          const double d = Dp[c * ldp + r];
          double val = pa * d;
          if (useB) val += bi * Acc[r * NCP + c];
          val += uu * (ms * Tsm[q * MAXC + c]);
          double o = a.cA[c] * val + a.cV[c] * d;
          if (P2) o += a.cP[c] * p2v[c];
          a.out[c * n_pad + p0 + r] = o;
          const double y2 = (a.epi == EPI_S) ? uu : (a.use_par_p2 == 2) ? d : (a.use_par_p2 == 1) ? p2v[c] : y2v[c];
          ep[c] = fma(o, y2, ep[c]);
        }
      }
    }
    if (useB) {
      bar_epi<PNE>();                                // all reads of Acc, Dp[q&1] and the T row done
      // D of piece q+2 into Dp[q&1]: copies issued now, completed (and combined) at the next piece
      if (q + 2 < nseg) {
        if (et == 0) {
          issue_d(q + 2);
          if (!a.fuse_p) mbar_arrive(&accfree[q % nacc]);   // (fused: Acc stages P_old until finish_d)
        }
        pend = q + 2;
      } else if (et == 0) {
        mbar_arrive(&accfree[q % nacc]);
      }
    }
    if (!run_epi) {
      if (et == 0 && q < 8) TR(37 + q);
      continue;
    }
    // per-cluster column sums: warp butterflies, then the warps in fixed order
#pragma unroll
    for (int c = 0; c < NCP; ++c) ep[c] = warp_sum(ep[c]);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < NCP; ++c) ered[ew * MAXC + c] = ep[c];
    bar_epi<PNE>();
    if (et < ncol) {
      double s = 0.0;
      for (int w = 0; w < PNE; ++w) s += ered[w * MAXC + et];
      if (a.epi == EPI_S) a.Sout[static_cast<int64_t>(i) * MAXC + et] = s;
      else a.dots[static_cast<int64_t>(i) * MAXC + et] = s;
    }
    bar_epi<PNE>();                                  // ered reuse
    if (et == 0 && q < 8) TR(37 + q);
  }
  // finaliser (last CTA; one epilogue warp per column)
  if (a.fin != FIN_NONE) {
    __threadfence();
    bar_epi<PNE>();
    if (et == 0) s_last = (atomicAdd(&a.st->ticket[a.fin], 1u) == gridDim.x - 1);
    bar_epi<PNE>();
    if (s_last) {
      __threadfence();
      fin_alpha_trace_body(a.fin, a.st, a.dots, a.L.n_c, ncol, a.alpha_hist, a.hist_stride, PNE, PWE);
      bar_epi<PNE>();
      if (et == 0) a.st->ticket[a.fin] = 0;
    }
  }
  if (et == 0) {
    TR(45);
    long long clk_end = 0;
    TCLK(clk_end);
    TRV(47, clk_end - clk_start);
  }
}

// --------------------------------------------------------------------------------------- host
bool plan_packed_apply(int ld_max, int ncol, bool f32, int seg_max, int lr_nc, ApplyArgs& a) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
    optin = 227 * 1024;
  a.nt8 = (ncol - 1 + 7) / 8;
  if (a.nt8 < 1) a.nt8 = 1;
  if (a.nt8 > 2 || ld_max > 512) return false;
  a.mtmax = (ld_max <= 128) ? 2 : (ld_max <= 256) ? 4 : 8;
  a.f32 = f32 ? 1 : 0;
  a.ld_max = ld_max;
  const int es = f32 ? 4 : 8;
  const int pne = 7;
  const size_t budget = static_cast<size_t>(optin) - 8192;   // static shared memory + margin
  // options in order of preference, the first that keeps >= 4 ring slots: a second Acc buffer (the
  // MMA warps run a piece ahead of the epilogue) and the staged M' rows (bulk copies, 16-byte rows)
  const int64_t mst_need = static_cast<int64_t>(seg_max) * lr_nc;
  const bool mst_ok = (lr_nc % 2) == 0;                        // (staged M' rows: 813 vs 809 evals/s at C3)
  const int opts[4][2] = {{2, 1}, {1, 1}, {2, 0}, {1, 0}};
  int ns = 0, nacc = 1, mst = 0;
  for (int o = 0; o < 5; ++o) {
    const int na = o < 4 ? opts[o][0] : 1, ms = o < 4 ? opts[o][1] : 0;
    if (ms && !mst_ok) continue;
    const PackSmem fixed = pack_smem(0, es, ld_max, a.nt8, pne, seg_max, na, ms ? mst_need : 0);
    if (fixed.total >= budget) continue;
    const int n = static_cast<int>(std::min<size_t>(MAX_NSTAGE, (budget - fixed.total) / (static_cast<size_t>(CHUNK) * 64 * es)));
    if (n >= 4 || (o == 4 && n >= 2)) { ns = n; nacc = na; mst = ms; break; }
  }
  if (ns < 2) return false;
  a.nacc = nacc;
  a.mst = mst;
  // S rows through the ring: off — with the thin-row split the stream needs all ring slots from the
  // start (C3, 3 A/B pairs: 814 vs 798 evals/s, 57.5 vs 58.9 us per apply without the staging)
  a.lr_stage_s = 0;
  a.slot_tiles = CHUNK;
  a.nstage = ns;
  a.smem = pack_smem(ns, es, ld_max, a.nt8, pne, seg_max, nacc, mst ? mst_need : 0).total;
  return true;
}

template <int NM, int MT, int N8, typename TB>
static void launch_pk(const ApplyArgs& a, cudaStream_t s) {
  // 16 or 13 warps (<= 4 per SM sub-partition: 128 registers), one CTA per SM
  constexpr int NE = 7;
  auto k = apply_packed_kernel<NM, MT, N8, TB, NE>;
  smem_optin(reinterpret_cast<const void*>(k));
  k<<<a.grid, (NM + NE + 1) * 32, a.smem, s>>>(a);
}

#ifdef NUGPR_TRACE_APPLY
static long long g_trace_count = 0, g_trace_at = -1;
#endif

void launch_apply_packed(const ApplyArgs& a, cudaStream_t s) {
#ifdef NUGPR_TRACE_APPLY
  if (g_trace_at < 0) { const char* e = getenv("NUGPR_TRACE_AT"); g_trace_at = e ? atoll(e) : 1LL << 60; }
  const bool tr = g_trace_count++ == g_trace_at;
  if (tr) {
    const int one = 1;
    void* tp = nullptr;
    cudaGetSymbolAddress(&tp, g_apply_trace);
    cudaMemsetAsync(tp, 0, sizeof(g_apply_trace), s);
    cudaMemcpyToSymbolAsync(g_apply_trace_on, &one, sizeof(int), 0, cudaMemcpyHostToDevice, s);
  }
#endif
#define NUGPR_PK(MT)                                                        \
  do {                                                                      \
    if (a.nt8 == 1) {                                                       \
      if (a.f32) launch_pk<8, MT, 1, float>(a, s); else launch_pk<8, MT, 1, double>(a, s); \
    } else {                                                                \
      launch_pk<8, MT, 2, double>(a, s);                                    \
    }                                                                       \
  } while (0)
  if (a.mtmax == 2) NUGPR_PK(2);
  else if (a.mtmax == 4) NUGPR_PK(4);
  else NUGPR_PK(8);
#undef NUGPR_PK
#ifdef NUGPR_TRACE_APPLY
  if (tr) { const int zero = 0; cudaMemcpyToSymbolAsync(g_apply_trace_on, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, s); }
#endif
  note_launch(); post_launch("apply_packed_kernel");
}

#ifdef NUGPR_TRACE_APPLY
extern "C" __attribute__((visibility("default"))) int nugpr_debug_apply_trace(unsigned long long* dst) {
  return cudaMemcpyFromSymbol(dst, g_apply_trace, sizeof(g_apply_trace)) == cudaSuccess ? 0 : 1;
}
#endif

}  // namespace nugpr
