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
//    no separate low-rank launch (the fused first apply also forms S(P_new) = S(R) + beta S(P_old)).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "cg_fin.cuh"
#include "common.cuh"
#include "kernels_decl.h"
#include "tma.cuh"

namespace nugpr {

constexpr int PNM = 8;                 // MMA warps (warp w owns the output m-tiles w, w+8, ...)
constexpr int PWE = PNM;               // first epilogue warp
constexpr int PNE_MAX = 7;             // epilogue / prologue warps: 7 (ld <= 256) or 4 (ld <= 512), register budget
constexpr int PLDP = 12;               // Dp row: 8 probe columns (conflict-free B fragments), y at slot 8
constexpr int TQ = 4;                  // pieces per reduction pass of the low-rank rows
constexpr int MAX_SEG_T = 8;           // pieces whose low-rank rows are formed from the staged S chunks

__device__ __forceinline__ void dmma_pk(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int PNE>
__device__ __forceinline__ void bar_epi() { asm volatile("bar.sync 2, %0;" ::"r"(PNE * 32) : "memory"); }

template <typename TB>
__device__ __forceinline__ double ldA(const TB* p) { return static_cast<double>(*p); }

// Shared-memory plan (host and device agree): ring | Dp[2] | Acc | Tsm
struct PackSmem {
  size_t ring, dp, acc, tsm, total;
};
__host__ __device__ inline PackSmem pack_smem(int slot_tiles, int nstage, int esize, int ld_max, int nt8, int seg_max) {
  PackSmem p;
  const size_t ncp = 1 + 8 * static_cast<size_t>(nt8);
  p.ring = 0;
  size_t o = static_cast<size_t>(nstage) * slot_tiles * 64 * esize;
  o = (o + 127) / 128 * 128;
  p.dp = o;
  o += 2 * static_cast<size_t>(nt8) * ld_max * PLDP * sizeof(double);
  p.acc = o;
  o += static_cast<size_t>(ld_max) * ncp * sizeof(double);
  p.tsm = o;
  o += (static_cast<size_t>(seg_max) * MAXC + (PNM + PNE_MAX) * TQ * 16) * sizeof(double);   // T rows + per-warp partials
  p.total = o;
  return p;
}

// The low-rank rows T_q = M'[row(q), :] S(D) need, per CTA, all n_c S rows (128 B each; with S(P_old)
// for the fused apply) and the CTA's M' rows.  They are staged through the still empty ring in chunks
// of JC rows of S together with the matching JC-wide segments of the M' rows (TMA path: n_c even and
// at most MAX_SEG_T pieces); JC is the same on every CTA of a launch.
__device__ __forceinline__ bool lr_tma(const ApplyArgs& a, int nseg) {
  return (a.lr_nc % 2) == 0 && nseg <= MAX_SEG_T;
}
__device__ __forceinline__ int lr_chunk_rows(const ApplyArgs& a, int esize) {
  const long ring_bytes = static_cast<long>(a.nstage) * a.slot_tiles * 64 * esize;
  const long per_row = (a.fuse_p ? 2 : 1) * MAXC * 8 + MAX_SEG_T * 8;   // S (+ S(P_old)) + M' segments
  return static_cast<int>(ring_bytes / per_row) & ~1;
}

// Warp-specialised persistent apply: 8 MMA warps stream the CTA's tile blocks, 4 epilogue warps form
// the next piece's D and run the previous piece's epilogue (and the split-cluster combine, the
// low-rank rows, the finaliser), 1 warp drives the TMA ring.  Handshakes (mbarriers):
//   full / empty [ring]        producer <-> MMA warps (one tile block per slot)
//   dready[2]                  epilogue -> MMA (D of piece q formed in Dp[q&1])
//   accready / accfree         MMA -> epilogue (block products of piece q in Acc; Dp[q&1] is free
//                              again) / epilogue -> MMA (Acc consumed)
template <int MTMAX, int NT8, typename TB, int PNE>
__global__ void __launch_bounds__((PNM + PNE + 1) * 32, 1) apply_packed_kernel(const __grid_constant__ ApplyArgs a) {
  constexpr int NCP = 1 + 8 * NT8;               // y + probe columns held per row
  constexpr int PWP = PNM + PNE;                 // the TMA producer warp
  if (a.gate && !a.st->any_active) return;
  const int b = blockIdx.x;
  const int s_lo = a.L.seg0[b], s_hi = a.L.seg0[b + 1];
  const int nseg = s_hi - s_lo;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t empty[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t dready[2], accready, accfree, tfull, tempty;
  __shared__ double ered[PNE_MAX * MAXC];
  __shared__ double cb[2 * MAXC];
  __shared__ int s_last;
  const PackSmem L_ = pack_smem(a.slot_tiles, a.nstage, static_cast<int>(sizeof(TB)), a.ld_max, NT8, a.L.seg_max);
  TB* ring = reinterpret_cast<TB*>(smraw + L_.ring);
  double* Dpb = reinterpret_cast<double*>(smraw + L_.dp);   // [2][NT8][ld_max][PLDP]
  double* Acc = reinterpret_cast<double*>(smraw + L_.acc);  // [ld_max][NCP] block products of a piece
  double* Tsm = reinterpret_cast<double*>(smraw + L_.tsm);  // [seg_max][MAXC], then partials
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n_pad = a.L.n_pad;
  const int ncol = a.ncol;
  const EvalParams* P = a.prm;
  const int par = a.st->par;
  const TB* B = (sizeof(TB) == 4) ? reinterpret_cast<const TB*>(P->B32) : reinterpret_cast<const TB*>(P->B);
  const bool useB = (P->B != nullptr);
  const int nstage = a.nstage, slot_tiles = a.slot_tiles;
  const int dpstride = NT8 * a.ld_max * PLDP;                // one Dp buffer
  const int ldD = a.ld_max * PLDP;                           // n8-tile stride within a buffer
  const double* Pold = a.fuse_p ? a.Pbuf[par] : nullptr;
  double* Pnew = a.fuse_p ? a.Pbuf[par ^ 1] : nullptr;
  const double* P2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.P2;
  const double* Y2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.Y2;
  const double* Dv = a.fuse_p ? Pnew : a.D;                  // the apply's input vector D (fused: P_new)
  if (tid == 0) {
    for (int s_ = 0; s_ < nstage; ++s_) { mbar_init(&full[s_], 1); mbar_init(&empty[s_], PNM); }
    for (int k = 0; k < 2; ++k) mbar_init(&dready[k], 1);
    mbar_init(&accready, PNM);
    mbar_init(&accfree, 1);
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 1);
    fence_mbar_init();
  }
  if (tid < MAXC) {
    cb[tid] = (tid < ncol) ? a.st->beta[tid] : 0.0;
    cb[MAXC + tid] = (tid < ncol) ? static_cast<double>(a.st->active[tid]) : 0.0;
  }
  __syncthreads();

  if (wid == PWP) {
    // ================================ TMA producer ================================
    if (lane == 0) {
      // first, ahead of the block stream: the M' rows of this CTA's pieces (the consumers' low-rank
      // rows read them right away; behind the stream they would wait in the DRAM queues)
      if ((a.lr_nc & 1) == 0)                        // (bulk prefetch: 16-byte aligned rows)
        for (int q = 0; q < nseg; ++q)
          tma_prefetch_l2(P->Mp + static_cast<int64_t>(a.lr_row0 + a.L.segs[s_lo + q].blk) * a.lr_nc,
                          static_cast<uint32_t>(a.lr_nc) * 8u);
      // the S rows of the low-rank term (and S(P_old) for the fused apply) and the M' row segments
      // staged through the still empty ring in chunks of JC rows, before the block stream starts
      if (lr_tma(a, nseg)) {
        const int JC = lr_chunk_rows(a, static_cast<int>(sizeof(TB)));
        double* ringd = reinterpret_cast<double*>(ring);
        int k = 0;
        for (int j0 = 0; j0 < a.lr_nc; j0 += JC, ++k) {
          if (k > 0) mbar_wait(&tempty, static_cast<uint32_t>((k - 1) & 1));
          const int jn = min(JC, a.lr_nc - j0);
          const uint32_t bytes = static_cast<uint32_t>(jn) * (MAXC * 8u);
          const uint32_t mbytes = static_cast<uint32_t>(jn) * 8u;
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&tfull, bytes * (a.fuse_p ? 2u : 1u) + mbytes * nseg);
          tma_load_1d(ringd, a.S_D + static_cast<int64_t>(j0) * MAXC, bytes, &tfull);
          if (a.fuse_p) tma_load_1d(ringd + JC * MAXC, a.SPbuf[par] + static_cast<int64_t>(j0) * MAXC, bytes, &tfull);
          double* mseg = ringd + (a.fuse_p ? 2 : 1) * JC * MAXC;
          for (int q = 0; q < nseg; ++q)
            tma_load_1d(mseg + q * JC, P->Mp + static_cast<int64_t>(a.lr_row0 + a.L.segs[s_lo + q].blk) * a.lr_nc + j0,
                        mbytes, &tfull);
        }
        mbar_wait(&tempty, static_cast<uint32_t>((k - 1) & 1));   // ring free again
      }
      uint32_t pseq = 0;
      for (int q = 0; q < nseg; ++q) {
        const SegDesc sd = a.L.segs[s_lo + q];
        const int i = sd.blk;
        const int ld = a.L.ld[i], mt = ld >> 3;
        const int64_t p0 = a.L.poff[i];
        // warm L2 with this piece's epilogue inputs and the next piece's D inputs (plain loads later)
        const uint32_t cbytes = static_cast<uint32_t>(ld) * 8u;
        tma_prefetch_l2(a.u + p0, cbytes);
        for (int c = 0; c < ncol; ++c) {
          if (P2) tma_prefetch_l2(P2 + c * n_pad + p0, cbytes);
          if (a.epi == EPI_DOT && Y2 && Y2 != P2) tma_prefetch_l2(Y2 + c * n_pad + p0, cbytes);
        }
        if (q + 1 < nseg) {
          const int i1 = a.L.segs[s_lo + q + 1].blk;
          const int64_t p1 = a.L.poff[i1];
          const uint32_t cb1 = static_cast<uint32_t>(a.L.ld[i1]) * 8u;
          for (int c = 0; c < ncol; ++c) {
            tma_prefetch_l2(a.D + c * n_pad + p1, cb1);
            if (a.fuse_p) tma_prefetch_l2(Pold + c * n_pad + p1, cb1);
          }
        }
        if (!useB) continue;
        // one chunk per tile block of the piece, in storage order (s-major, g ascending)
        const TB* Bi = B + a.L.pboff[i];
        const int ns = pk_ns(mt);
        int sb = 0, gb = 0;
        for (int k = 0; k < sd.k0; ++k) { if (++gb == ns) { ++sb; gb = sb; } }
        for (int k = sd.k0; k < sd.k1; ++k, ++pseq) {
          const int s_ = static_cast<int>(pseq % nstage);
          const uint32_t use = pseq / nstage;
          if (use > 0) mbar_wait(&empty[s_], (use - 1) & 1u);
          const int nt = pk_blk_size(gb, sb, mt);
          const uint32_t bytes = static_cast<uint32_t>(nt) * 64u * static_cast<uint32_t>(sizeof(TB));
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full[s_], bytes);
          tma_load_1d(ring + static_cast<int64_t>(s_) * slot_tiles * 64,
                      Bi + static_cast<int64_t>(pk_blk_off(gb, sb, mt)) * 64, bytes, &full[s_]);
          if (++gb == ns) { ++sb; gb = sb; }
        }
      }
    }
    return;
  }

  // ===================== consumer prologue (MMA + epilogue warps together) =====================
  constexpr int NCW = PNM + PNE;                     // consumer warps
  const int ct = tid;                                // 0 .. 32 NCW - 1
  auto bar_cons_all = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory"); };
  // form D of piece q in Dp[q&1] (fused: D = R + beta o P_old for the active columns, P_new written by
  // part 0), coalesced over the rows of each column; nthr threads starting at thread t0
  auto form_d = [&](int q, int t0, int nthr) {
    const SegDesc sd = a.L.segs[s_lo + q];
    const int i = sd.blk, ld = a.L.ld[i];
    const int64_t p0 = a.L.poff[i];
    double* Dp = Dpb + (q & 1) * dpstride;
    constexpr int U = 4;                             // elements per thread in flight
    const int tot = ld * ncol;
    for (int base = t0; base < tot; base += U * nthr) {
      double v[U], po[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * nthr;
        v[u] = 0.0;
        po[u] = 0.0;
        if (idx < tot) {
          const int c = idx / ld, k = idx - c * ld;
          const int64_t gi = c * n_pad + p0 + k;
          v[u] = __ldg(a.D + gi);
          if (a.fuse_p) po[u] = __ldg(Pold + gi);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * nthr;
        if (idx < tot) {
          const int c = idx / ld, k = idx - c * ld;
          double x = v[u];
          if (a.fuse_p) {
            x = (cb[MAXC + c] != 0.0) ? x + cb[c] * po[u] : po[u];
            if (sd.part == 0) Pnew[c * n_pad + p0 + k] = x;
          }
          if (useB) Dp[(c == 0) ? k * PLDP + 8 : ((c - 1) >> 3) * ldD + k * PLDP + ((c - 1) & 7)] = x;
        }
      }
    }
  };
  // low-rank rows T_q = M'[row(q), :] S(D) for every piece q of this CTA, with S read once per CTA in
  // coalesced rows: thread ct owns column c = ct % 16 of the S rows j = ct/16 + 2 NCW k (8 in flight),
  // times M'[row(q), j] for TQ pieces per pass; the row-offsets of each column are summed in fixed
  // order (lane pairs, then warps) — the same decomposition on every CTA, so a cluster's T has the
  // same bits wherever it is formed.  All consumer warps take part, before the pipeline starts.
  {
    const double* SPo = a.fuse_p ? a.SPbuf[par] : nullptr;
    const double* Mp = P->Mp;
    const int nc = a.lr_nc;
    const int c = ct & 15, j0 = ct >> 4;
    const bool cact = c < ncol;
    const double bc = cb[c], ac = cb[MAXC + c];
    double* Tpart = Tsm + a.L.seg_max * MAXC;       // [NCW][TQ][16]
    // (TMA path: the S rows and the M' row segments arrive through the ring in chunks of JC rows —
    //  the same chunking on every CTA of a launch; in each chunk a thread takes rows j0, j0 + NJ, ...)
    constexpr int NJ = 2 * NCW;
    double t[MAX_SEG_T];
#pragma unroll
    for (int qq = 0; qq < MAX_SEG_T; ++qq) t[qq] = 0.0;
    const bool tma_path = lr_tma(a, nseg);
    if (tma_path) {
      const int JC = lr_chunk_rows(a, static_cast<int>(sizeof(TB)));
      const double* ringd = reinterpret_cast<const double*>(ring);
      const double* mseg = ringd + (a.fuse_p ? 2 : 1) * JC * MAXC;
      int k = 0;
      for (int jc = 0; jc < nc; jc += JC, ++k) {
        const int jn = min(JC, nc - jc);
        mbar_wait(&tfull, static_cast<uint32_t>(k & 1));
        for (int jj = j0; jj < jn; jj += NJ) {
          double x = 0.0;
          if (cact) {
            x = ringd[jj * MAXC + c];
            if (a.fuse_p) {
              const double y = ringd[(JC + jj) * MAXC + c];
              x = (ac != 0.0) ? x + bc * y : y;
            }
          }
#pragma unroll
          for (int qq = 0; qq < MAX_SEG_T; ++qq)
            if (qq < nseg) t[qq] = fma(mseg[qq * JC + jj], x, t[qq]);
        }
        bar_cons_all();
        if (ct == 0) mbar_arrive(&tempty);
      }
    }
    // (global path: n_c odd, or more than MAX_SEG_T pieces, e.g. C5's many clusters per CTA)
    for (int qb = tma_path ? nseg : 0; qb < nseg; ++qb) {
      const double* Mr = Mp + static_cast<int64_t>(a.lr_row0 + a.L.segs[s_lo + qb].blk) * nc;
      double tv = 0.0;
      for (int j = j0; j < nc; j += NJ) {
        double x = 0.0;
        if (cact) {
          x = a.S_D[static_cast<int64_t>(j) * MAXC + c];
          if (a.fuse_p) {
            const double y = SPo[static_cast<int64_t>(j) * MAXC + c];
            x = (ac != 0.0) ? x + bc * y : y;
          }
        }
        tv = fma(__ldg(Mr + j), x, tv);
      }
      tv += __shfl_xor_sync(0xffffffffu, tv, 16);
      if (lane < 16) Tpart[wid * 16 + lane] = tv;
      bar_cons_all();
      if (ct < 16) {
        double acc_ = 0.0;
        for (int w = 0; w < NCW; ++w) acc_ += Tpart[w * 16 + ct];
        Tsm[qb * MAXC + ct] = acc_;
      }
      bar_cons_all();
    }
#pragma unroll
    for (int qq = 0; qq < MAX_SEG_T; ++qq) t[qq] += __shfl_xor_sync(0xffffffffu, t[qq], 16);
#pragma unroll
    for (int qb = 0; qb < MAX_SEG_T; qb += TQ) {
      if (!tma_path || qb >= nseg) break;
      if (lane < 16)
#pragma unroll
        for (int qq = 0; qq < TQ; ++qq) Tpart[(wid * TQ + qq) * 16 + lane] = t[qb + qq];
      bar_cons_all();
      const int nq = min(TQ, min(nseg, MAX_SEG_T) - qb);
      if (ct < nq * 16) {
        const int qq = ct >> 4, cc = ct & 15;
        double acc_ = 0.0;
        for (int w = 0; w < NCW; ++w) acc_ += Tpart[(w * TQ + qq) * 16 + cc];
        Tsm[(qb + qq) * MAXC + cc] = acc_;
      }
      bar_cons_all();
    }
    if (a.fuse_p && b == 0) {
      // S(P_new) = S(R) + beta o S(P_old) (active columns; S is linear) for the next iteration
      for (int idx = ct; idx < nc * ncol; idx += NCW * 32) {
        const int j = idx / ncol, cc = idx - j * ncol;
        const double x = a.S_D[static_cast<int64_t>(j) * MAXC + cc], y = SPo[static_cast<int64_t>(j) * MAXC + cc];
        a.SPbuf[par ^ 1][static_cast<int64_t>(j) * MAXC + cc] = (cb[MAXC + cc] != 0.0) ? x + cb[cc] * y : y;
      }
    }
  }
  if (useB) {                                       // D of the first two pieces (both Dp buffers)
    for (int q = 0; q < min(2, nseg); ++q) form_d(q, ct, NCW * 32);
    bar_cons_all();
  }

  if (wid < PNM) {
    // ================================ MMA warps ================================
    if (!useB) return;                               // no block term: the epilogue warps do everything
    const int qr = lane >> 2, qc = lane & 3;
    const int offD0 = swz(qr, qc), offD1 = swz(qr, 4 + qc);    // A = T:    T[qr][h4 + qc]
    const int offT0 = swz(qc, qr), offT1 = swz(4 + qc, qr);    // A = T^T:  T[h4 + qc][qr]
    uint32_t seq = 0;
    for (int q = 0; q < nseg; ++q) {
      const SegDesc sd = a.L.segs[s_lo + q];
      const int mt = a.L.ld[sd.blk] >> 3;
      const double* Dp = Dpb + (q & 1) * dpstride;
      mbar_wait(&dready[q & 1], static_cast<uint32_t>((q >> 1) & 1));
      double acc[NT8][2][MTMAX], accy[MTMAX];
#pragma unroll
      for (int j = 0; j < MTMAX; ++j) {
        accy[j] = 0.0;
#pragma unroll
        for (int n = 0; n < NT8; ++n) { acc[n][0][j] = 0.0; acc[n][1][j] = 0.0; }
      }
      const int ns = pk_ns(mt);
      int sb = 0, gb = 0;
      for (int k = 0; k < sd.k0; ++k) { if (++gb == ns) { ++sb; gb = sb; } }
      for (int k = sd.k0; k < sd.k1; ++k, ++seq) {
        const int s_ = static_cast<int>(seq % nstage);
        const TB* blk = ring + static_cast<int64_t>(s_) * slot_tiles * 64;
        const int h = pk_h(gb, mt), w = pk_h(sb, mt);
        const bool diag = gb == sb;
        mbar_wait(&full[s_], (seq / nstage) & 1u);
        // full 8x8-tile block: warp w does, for k = 0..7, the direct tile (w, k) (k <= w on the
        // diagonal) and the transposed tile (k, w) (k > w on the diagonal) with four independent
        // accumulator chains (direct / transposed x even / odd k)
        auto full_block = [&](auto diag_c) {
          constexpr bool DG = decltype(diag_c)::value;
          double d0[2][NT8], d1[2][NT8], dy[2] = {0.0, 0.0};
          double t0[2][NT8], t1[2][NT8], ty[2] = {0.0, 0.0};
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int n = 0; n < NT8; ++n) { d0[e][n] = 0.0; d1[e][n] = 0.0; t0[e][n] = 0.0; t1[e][n] = 0.0; }
          const int rowK = 64 * sb, rowI = 64 * gb;          // first D row of the block's columns / rows
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int e = kk & 1;
            if (!DG || kk <= wid) {
              const int pos = DG ? 8 * kk - kk * (kk - 1) / 2 + (wid - kk) : 8 * kk + wid;
              const TB* tp = blk + pos * 64;
              const double a0 = ldA(tp + offD0), a1 = ldA(tp + offD1);
              const double* dr = Dp + (rowK + 8 * kk) * PLDP;
#pragma unroll
              for (int n = 0; n < NT8; ++n) {
                dmma_pk(d0[e][n], d1[e][n], a0, dr[n * ldD + qc * PLDP + qr]);
                dmma_pk(d0[e][n], d1[e][n], a1, dr[n * ldD + (4 + qc) * PLDP + qr]);
              }
              dy[e] = fma(a0, dr[qc * PLDP + 8], dy[e]);
              dy[e] = fma(a1, dr[(4 + qc) * PLDP + 8], dy[e]);
            }
            if (!DG || kk > wid) {
              const int pos = DG ? 8 * wid - wid * (wid - 1) / 2 + (kk - wid) : 8 * wid + kk;
              const TB* tp = blk + pos * 64;
              const double a0 = ldA(tp + offT0), a1 = ldA(tp + offT1);
              const double* dr = Dp + (rowI + 8 * kk) * PLDP;
#pragma unroll
              for (int n = 0; n < NT8; ++n) {
                dmma_pk(t0[e][n], t1[e][n], a0, dr[n * ldD + qc * PLDP + qr]);
                dmma_pk(t0[e][n], t1[e][n], a1, dr[n * ldD + (4 + qc) * PLDP + qr]);
              }
              ty[e] = fma(a0, dr[qc * PLDP + 8], ty[e]);
              ty[e] = fma(a1, dr[(4 + qc) * PLDP + 8], ty[e]);
            }
          }
#pragma unroll
          for (int j = 0; j < MTMAX; ++j) {
            if (j == gb) {                                    // direct: rows I = 8g + w
#pragma unroll
              for (int n = 0; n < NT8; ++n) { acc[n][0][j] += d0[0][n] + d0[1][n]; acc[n][1][j] += d1[0][n] + d1[1][n]; }
              accy[j] += dy[0] + dy[1];
            }
            if (j == sb) {                                    // transposed: columns K = 8s + w
#pragma unroll
              for (int n = 0; n < NT8; ++n) { acc[n][0][j] += t0[0][n] + t0[1][n]; acc[n][1][j] += t1[0][n] + t1[1][n]; }
              accy[j] += ty[0] + ty[1];
            }
          }
        };
        if (h == 8 && w == 8) {
          if (diag) full_block(std::true_type());
          else full_block(std::false_type());
        } else {
          // edge block (the last block row / column of a cluster whose ld is not a multiple of 64)
          double x0[NT8], x1[NT8], xy = 0.0;
#pragma unroll
          for (int n = 0; n < NT8; ++n) { x0[n] = 0.0; x1[n] = 0.0; }
          if (wid < w) {                                      // transposed: column b = wid
            const int bcol = wid;
            const int cbase = diag ? bcol * h - bcol * (bcol - 1) / 2 - bcol : bcol * h;   // tile (a, b) at cbase + a
            for (int aa = diag ? bcol + 1 : 0; aa < h; ++aa) {
              const TB* tp = blk + (cbase + aa) * 64;
              const double a0 = ldA(tp + offT0), a1 = ldA(tp + offT1);
              const double* dr = Dp + (64 * gb + 8 * aa) * PLDP;
#pragma unroll
              for (int n = 0; n < NT8; ++n) {
                dmma_pk(x0[n], x1[n], a0, dr[n * ldD + qc * PLDP + qr]);
                dmma_pk(x0[n], x1[n], a1, dr[n * ldD + (4 + qc) * PLDP + qr]);
              }
              xy = fma(a0, dr[qc * PLDP + 8], xy);
              xy = fma(a1, dr[(4 + qc) * PLDP + 8], xy);
            }
#pragma unroll
            for (int j = 0; j < MTMAX; ++j)
              if (j == sb) {
#pragma unroll
                for (int n = 0; n < NT8; ++n) { acc[n][0][j] += x0[n]; acc[n][1][j] += x1[n]; x0[n] = 0.0; x1[n] = 0.0; }
                accy[j] += xy;
                xy = 0.0;
              }
          }
          if (wid < h) {                                      // direct: row a = wid
            const int arow = wid;
            const int b_hi = diag ? arow : w - 1;
            for (int bb = 0; bb <= b_hi; ++bb) {
              const int pos = diag ? bb * h - bb * (bb - 1) / 2 + (arow - bb) : bb * h + arow;
              const TB* tp = blk + pos * 64;
              const double a0 = ldA(tp + offD0), a1 = ldA(tp + offD1);
              const double* dr = Dp + (64 * sb + 8 * bb) * PLDP;
#pragma unroll
              for (int n = 0; n < NT8; ++n) {
                dmma_pk(x0[n], x1[n], a0, dr[n * ldD + qc * PLDP + qr]);
                dmma_pk(x0[n], x1[n], a1, dr[n * ldD + (4 + qc) * PLDP + qr]);
              }
              xy = fma(a0, dr[qc * PLDP + 8], xy);
              xy = fma(a1, dr[(4 + qc) * PLDP + 8], xy);
            }
#pragma unroll
            for (int j = 0; j < MTMAX; ++j)
              if (j == gb) {
#pragma unroll
                for (int n = 0; n < NT8; ++n) { acc[n][0][j] += x0[n]; acc[n][1][j] += x1[n]; }
                accy[j] += xy;
              }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s_]);
        if (++gb == ns) { ++sb; gb = sb; }
      }
      // y column: sum the 4 k-lanes of each row quad
#pragma unroll
      for (int j = 0; j < MTMAX; ++j) {
        accy[j] += __shfl_xor_sync(0xffffffffu, accy[j], 1);
        accy[j] += __shfl_xor_sync(0xffffffffu, accy[j], 2);
      }
      if (q > 0) mbar_wait(&accfree, static_cast<uint32_t>((q - 1) & 1));
#pragma unroll
      for (int j = 0; j < MTMAX; ++j) {
        const int mtj = wid + j * PNM;
        if (mtj < mt) {
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
      if (lane == 0) mbar_arrive(&accready);
    }
    return;
  }

  // ================================ epilogue warps ================================
  const int et = tid - PWE * 32;                     // 0 .. 32 PNE - 1
  const int ew = wid - PWE;
  if (useB && et == 0)
    for (int q = 0; q < min(2, nseg); ++q) mbar_arrive(&dready[q]);
  for (int q = 0; q < nseg; ++q) {
    const SegDesc sd = a.L.segs[s_lo + q];
    const int i = sd.blk, ld = a.L.ld[i];
    const int64_t p0 = a.L.poff[i];
    if (!useB) {
      form_d(q, et, PNE * 32);                       // (fused apply without a block term: P_new only)
      bar_epi<PNE>();
    }
    if (useB) {
      mbar_wait(&accready, static_cast<uint32_t>(q & 1));
      // the MMA warps are done with Dp[q&1]: D of piece q+2 goes there while they stream piece q+1
      if (q + 2 < nseg) {
        form_d(q + 2, et, PNE * 32);
        bar_epi<PNE>();
        if (et == 0) mbar_arrive(&dready[q & 1]);
      }
      // split cluster: publish this part's block products; the last part sums all parts in order
      if (sd.nparts > 1) {
        double* base = a.split_part + sd.spoff + static_cast<int64_t>(sd.part) * ld * NCP;
        for (int idx = et; idx < ld * NCP; idx += PNE * 32) base[idx] = Acc[idx];
        __threadfence();
        bar_epi<PNE>();
        if (et == 0) s_last = (atomicAdd(&a.split_ticket[sd.tick], 1u) == static_cast<unsigned>(sd.nparts - 1));
        bar_epi<PNE>();
        if (!s_last) {
          if (et == 0) mbar_arrive(&accfree);
          continue;
        }
        __threadfence();
        const double* all = a.split_part + sd.spoff;
        const int64_t pst = static_cast<int64_t>(ld) * NCP;
        for (int base = et; base < ld * NCP; base += 2 * PNE * 32) {
          double v[2][MAX_PARTS];
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int pp = 0; pp < MAX_PARTS; ++pp) {
              const int idx = base + u * PNE * 32;
              v[u][pp] = (idx < ld * NCP && pp < sd.nparts) ? __ldcg(all + pp * pst + idx) : 0.0;
            }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int idx = base + u * PNE * 32;
            if (idx < ld * NCP) {
              double acc_ = v[u][0];
              for (int pp = 1; pp < sd.nparts; ++pp) acc_ += v[u][pp];
              Acc[idx] = acc_;
            }
          }
        }
        if (et == 0) a.split_ticket[sd.tick] = 0u;
        bar_epi<PNE>();
      }
    } else if (sd.part != 0) {
      continue;                                      // no block term: part 0 holds the whole result
    }
    // epilogue: thread et owns rows r = et, et + 128, ... (coalesced over r for every column c)
    double ep[NCP];
#pragma unroll
    for (int c = 0; c < NCP; ++c) ep[c] = 0.0;
    {
      const double bi = P->b0 + P->b1 * a.jitter[i];
      const double pa = P->a, ms = P->mscale;
      const double* Tq = Tsm + q * MAXC;
      // loads of a row first (all columns in flight), then the arithmetic
      for (int r = et; r < ld; r += PNE * 32) {
        const double uu = __ldg(a.u + p0 + r);
        double dv[NCP], p2v[NCP], y2v[NCP];
#pragma unroll
        for (int c = 0; c < NCP; ++c) {
          const int64_t gi = c * n_pad + p0 + r;
          const bool on = c < ncol;
          dv[c] = on ? Dv[gi] : 0.0;
          p2v[c] = (on && P2) ? P2[gi] : 0.0;
          y2v[c] = (on && a.epi == EPI_DOT && a.use_par_p2 == 0) ? Y2[gi] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < NCP; ++c) {
          if (c >= ncol) continue;
          const double d = dv[c];
          double val = pa * d;
          if (useB) val += bi * Acc[r * NCP + c];
          val += uu * (ms * Tq[c]);
          double o = a.cA[c] * val + a.cV[c] * d;
          if (P2) o += a.cP[c] * p2v[c];
          a.out[c * n_pad + p0 + r] = o;
          const double y2 = (a.epi == EPI_S) ? uu : (a.use_par_p2 == 2) ? d : (a.use_par_p2 == 1) ? p2v[c] : y2v[c];
          ep[c] = fma(o, y2, ep[c]);
        }
      }
    }
    if (useB) {
      bar_epi<PNE>();                                     // all reads of Acc done
      if (et == 0) mbar_arrive(&accfree);
    }
    // per-cluster column sums: warp butterflies, then the 4 warps in fixed order
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
    bar_epi<PNE>();                                       // ered reuse
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
}

// --------------------------------------------------------------------------------------- host
bool plan_packed_apply(int ld_max, int ncol, bool f32, int seg_max, ApplyArgs& a) {
  // the ring slot holds one tile block (<= 64 tiles); at least 2 slots
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
  const size_t budget = static_cast<size_t>(optin) - 8192;   // static shared memory + margin
  for (int slot : {64}) {
    const PackSmem fixed = pack_smem(slot, 0, es, ld_max, a.nt8, seg_max);
    if (fixed.total >= budget) continue;
    const int ns = static_cast<int>(std::min<size_t>(MAX_NSTAGE, (budget - fixed.total) / (static_cast<size_t>(slot) * 64 * es)));
    if (ns >= 2) {
      a.slot_tiles = slot;
      a.nstage = ns;
      a.smem = pack_smem(slot, ns, es, ld_max, a.nt8, seg_max).total;
      return true;
    }
  }
  return false;
}

template <int MT, int N8, typename TB>
static void launch_pk(const ApplyArgs& a, cudaStream_t s) {
  constexpr int NE = (MT <= 4) ? 7 : 4;      // 16 or 13 warps: <= 4 per SM sub-partition (128 registers)
  auto k = apply_packed_kernel<MT, N8, TB, NE>;
  smem_optin(reinterpret_cast<const void*>(k));
  k<<<a.grid, (PNM + NE + 1) * 32, a.smem, s>>>(a);
}

void launch_apply_packed(const ApplyArgs& a, cudaStream_t s) {
#define NUGPR_PK(MT)                                                        \
  do {                                                                      \
    if (a.nt8 == 1) {                                                       \
      if (a.f32) launch_pk<MT, 1, float>(a, s); else launch_pk<MT, 1, double>(a, s); \
    } else {                                                                \
      launch_pk<MT, 2, double>(a, s);                                       \
    }                                                                       \
  } while (0)
  if (a.mtmax == 2) NUGPR_PK(2);
  else if (a.mtmax == 4) NUGPR_PK(4);
  else NUGPR_PK(8);
#undef NUGPR_PK
  note_launch(); post_launch("apply_packed_kernel");
}

}  // namespace nugpr
