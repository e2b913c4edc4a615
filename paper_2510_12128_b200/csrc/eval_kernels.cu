// eval_kernels.cu — rows A3-A7 of SURVEY §8(a): the fused multi-RHS apply of
// A = R^{-T} K''(theta) R^{-1} (Eq. 18-21, 23-25), the fused PCG update
// (PAPER.md:107-108, 124), the Pade trace (Eq. 9-10, 16), the SLQ
// log-det from the CG coefficients and the MLL assembly (Eq. 3).
//
// One evaluation = rhs_init -> { apply(A p) -> apply(Q(A) p) -> update }* -> spart(X) ->
// apply(A X) -> apply(3 A^2 X - 3 X, dotted with Z) -> final.  Every global reduction
// (S = W^T D, p^T q, r^T r, the trace dots) is written as per-tile partials and summed by
// the last CTA to finish, in fixed tile order: results are bit-reproducible.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels_decl.h"
#include "tma.cuh"
#include "tridiag.h"

namespace nugpr {

// Block-wide fixed-order reduction of NCP per-thread values -> out[0..NCP) (smem).
template <int NCP>
__device__ __forceinline__ void block_reduce_cols(double (&v)[NCP], double* sred, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < NCP; ++c) v[c] = warp_sum(v[c]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < NCP; ++c) sred[wid * NCP + c] = v[c];
  }
  __syncthreads();
  if (threadIdx.x < NCP) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += sred[w * NCP + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Last-CTA election (threadfence reduction pattern): true in every thread of the last CTA.
__device__ __forceinline__ bool last_cta(unsigned int* ticket) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// Deterministic total of column c of per-tile partials [n_tiles][MAXC]: called by a whole
// warp; lanes stride over tiles, then an xor-butterfly (every lane ends with the same bits).
__device__ __forceinline__ double col_total(const double* part, int n_tiles, int c) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int t = lane; t < n_tiles; t += 32) s += part[t * MAXC + c];
  return warp_sum(s);
}

// Column activity rule (PAPER.md:406 tol/max_iter, readings P3, P5; replay for parity).
__device__ __forceinline__ int is_active(const EvalParams* P, int c, int iters, double rr) {
  if (P->replay) return iters < P->replay_iters[c];
  if (iters >= P->max_iter) return 0;
  if (sqrt(rr) < P->tol) return 0;
  if (!(rr > 0.0)) return 0;
  return 1;
}

// ---------------------------------------------------------------------------------------
// CG finalisers.  Each runs in ONE CTA over the per-tile partials: in the last CTA of the
// kernel that wrote them (one GPU), or in fin_kernel after the PAR-2 exchange made the partials
// of every rank's clusters visible (same partial layout, same summation order => same bits).
// Warps w = 0..nw-1 stride over the columns.
__device__ void fin_init_body(CGState* st, const EvalParams* prm, const double* rr_part, int n_tiles, int ncol,
                              int nw) {
  __shared__ int act[MAXC], bd[MAXC];
  if (threadIdx.x < MAXC) bd[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid < nw) {
    for (int c = wid; c < MAXC; c += nw) {
      if (c < ncol) {
        const double tot = col_total(rr_part, n_tiles, c);
        if (lane == 0) {
          st->rr[c] = tot;
          st->rr0[c] = tot;
          st->alpha[c] = 0.0;
          st->beta[c] = 0.0;
          st->iters[c] = 0;
          st->t[c] = 0.0;
          act[c] = st->active[c] = isfinite(tot) ? is_active(prm, c, 0, tot) : 0;
          if (!isfinite(tot)) bd[c] = 1;
        }
      } else if (lane == 0) {
        st->active[c] = 0; st->iters[c] = 0; st->beta[c] = 0.0; st->alpha[c] = 0.0;
        act[c] = 0;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0, b = 0;
    for (int c = 0; c < ncol; ++c) { any |= act[c]; b |= bd[c]; }
    st->any_active = any;
    st->par = 0;
    st->hit_max = 0;
    st->breakdown = b;
    st->quad = 0.0;
  }
}

// FIN_ALPHA: alpha_c = r^T r / p^T q (active columns) + history; FIN_TRACE: quad (column 0) and the
// Pade trace terms t_j.  No block barrier inside (the DMMA apply calls it from its consumer warps).
__device__ __forceinline__ void fin_alpha_trace_body(int fin, CGState* st, const double* dots, int n_tiles,
                                                     int ncol, double* alpha_hist, int hist_stride, int nw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid >= nw) return;
  for (int c = wid; c < ncol; c += nw) {
    const double tot = col_total(dots, n_tiles, c);
    if (lane == 0) {
      if (fin == FIN_ALPHA) {
        if (st->active[c]) {
          const double al = st->rr[c] / tot;          // alpha = r^T r / p^T q
          if (!(tot > 0.0) || !isfinite(al)) {
            // breakdown: A is SPD in exact arithmetic, so p^T q <= 0 or a non-finite value means the
            // operator is not SPD at this theta or the inputs are not finite; freeze the column
            st->active[c] = 0;
            st->alpha[c] = 0.0;
            st->breakdown = 1;
          } else {
            st->alpha[c] = al;
            alpha_hist[c * hist_stride + st->iters[c]] = al;
          }
        }
      } else {  // FIN_TRACE
        if (c == 0) st->quad = tot; else st->t[c] = tot;
      }
    }
  }
}

// FIN_UPDATE: beta = r'^T r' / r^T r, history, iteration counters, freezing (readings P3, P5).
__device__ void fin_update_body(CGState* st, const EvalParams* P, const double* rr_part, int n_tiles, int ncol,
                                double* beta_hist, int hist_stride, unsigned long long cond, int nw) {
  __shared__ int act[MAXC];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int par = st->par;
  if (wid < nw) {
    for (int c = wid; c < ncol; c += nw) {
      const bool was = st->active[c] != 0;
      double tot = 0.0;
      if (was) tot = col_total(rr_part, n_tiles, c);
      if (lane == 0) {
        if (was) {
          const double be = tot / st->rr[c];
          st->beta[c] = be;
          beta_hist[c * hist_stride + st->iters[c]] = be;
          st->rr[c] = tot;
          st->iters[c] += 1;
          int na = is_active(P, c, st->iters[c], tot);
          if (!isfinite(tot)) { na = 0; st->breakdown = 1; }
          if (!na && !P->replay && st->iters[c] >= P->max_iter && !(sqrt(tot) < P->tol) && tot > 0.0)
            st->hit_max = 1;
          st->active[c] = na;
        }
        act[c] = st->active[c];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0;
    for (int c = 0; c < ncol; ++c) any |= act[c];
    st->any_active = any;
    st->par = par ^ 1;
    if (cond) cudaGraphSetConditional(cond, any ? 1u : 0u);
  }
}

// PAR-2 (cluster-sharded evaluation): the finaliser as its own single-CTA launch
// after the exchange of the partials.  FIN_UPDATE skips when no column is active (as update does).
__global__ void __launch_bounds__(NT) fin_kernel(int fin, CGState* st, const EvalParams* prm, const double* part,
                                                 int n_tiles, int ncol, double* hist, int hist_stride) {
  if (fin == FIN_INIT) {
    fin_init_body(st, prm, part, n_tiles, ncol, NT / 32);
  } else if (fin == FIN_UPDATE) {
    if (!st->any_active) return;
    fin_update_body(st, prm, part, n_tiles, ncol, hist, hist_stride, 0ull, NT / 32);
  } else {
    if (fin == FIN_ALPHA && !st->any_active) return;
    fin_alpha_trace_body(fin, st, part, n_tiles, ncol, hist, hist_stride, NT / 32);
  }
}

// Row r of the per-cluster lower triangular product c_i = Linv_i y_i (c = R^{-T} y):
// one fixed summation order, shared by rhs_init and cy_kernel so both give the same bits.
__device__ __forceinline__ double trmv_row(const double* Li, const double* ys, int ld, int r) {
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  int k = 0;
  for (; k + 3 <= r; k += 4) {
    c0 = fma(Li[static_cast<int64_t>(k) * ld + r], ys[k], c0);
    c1 = fma(Li[static_cast<int64_t>(k + 1) * ld + r], ys[k + 1], c1);
    c2 = fma(Li[static_cast<int64_t>(k + 2) * ld + r], ys[k + 2], c2);
    c3 = fma(Li[static_cast<int64_t>(k + 3) * ld + r], ys[k + 3], c3);
  }
  for (; k <= r; ++k) c0 = fma(Li[static_cast<int64_t>(k) * ld + r], ys[k], c0);
  return (c0 + c1) + (c2 + c3);
}

// c = R^{-T} y for all clusters (padded layout, zero on padding rows), computed once per
// numerical gradient and shared by its concurrent evaluations.
__global__ void __launch_bounds__(NT) cy_kernel(LayoutDev L, const double* Linv, const double* y, double* cy) {
  extern __shared__ double ys[];
  const TileDesc td = L.tiles[blockIdx.x];
  const int i = td.blk;
  const int ld = L.ld[i];
  const int64_t o = L.off[i], p0 = L.poff[i];
  const int b = static_cast<int>(L.off[i + 1] - o);
  for (int k = threadIdx.x; k < ld; k += NT) ys[k] = (k < b) ? y[o + k] : 0.0;
  __syncthreads();
  const double* Li = Linv + L.boff[i];
  for (int rl = threadIdx.x; rl < td.nrows; rl += NT) {
    const int r = td.row0 + rl;
    cy[p0 + r] = (r < b) ? trmv_row(Li, ys, ld, r) : 0.0;
  }
}

// ---------------------------------------------------------------------------------------
// rhs_init: RHS col 0 = c = Linv y (per-cluster lower trmv), cols 1..m = probes z_j;
// R = P_0 = RHS, X = 0; partials of r^T r and S(R); the last CTA initialises the CG state.
__global__ void __launch_bounds__(NT) rhs_init_kernel(RhsArgs a) {
  extern __shared__ double sm[];
  const int t = blockIdx.x;
  const TileDesc td = a.L.tiles[t];
  const int i = td.blk;
  const int ld = a.L.ld[i];
  const int64_t p0 = a.L.poff[i];
  const int64_t o = a.L.off[i];
  const int b = static_cast<int>(a.L.off[i + 1] - o);
  const int64_t n_pad = a.L.n_pad;
  const int64_t n = a.L.n;
  const int ncol = a.ncol;
  double* ys = sm;                      // ld
  double* sred = ys + ld;               // NT * MAXC
  double* outv = sred + NT * MAXC;      // MAXC
  for (int k = threadIdx.x; k < ld; k += NT) ys[k] = (k < b) ? a.y[o + k] : 0.0;
  __syncthreads();
  const double* Li = a.Linv + a.L.boff[i];
  double rr[MAXC], sr[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) { rr[c] = 0.0; sr[c] = 0.0; }
  for (int rl = threadIdx.x; rl < td.nrows; rl += NT) {
    const int r = td.row0 + rl;
    const int64_t g = p0 + r;
    const double uu = a.u[g];
    double cval = 0.0;
    if (a.cy) {
      cval = a.cy[g];
    } else if (r < b) {
      cval = trmv_row(Li, ys, ld, r);
    }
    if (a.cy_out) a.cy_out[g] = cval;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      if (c >= ncol) break;
      double v;
      if (c == 0) v = cval;
      else if (r >= b) v = 0.0;
      else v = a.probes ? a.probes[static_cast<int64_t>(c - 1) * a.n_glob + a.pos0 + o + r]
                         : probe_value(a.seed, c - 1, a.pos0 + o + r);
      const int64_t gi = c * n_pad + g;
      a.RHS[gi] = v;
      a.R[gi] = v;
      a.P0[gi] = v;
      a.X[gi] = 0.0;
      rr[c] += v * v;
      sr[c] += uu * v;
    }
  }
  block_reduce_cols<MAXC>(rr, sred, outv);
  if (threadIdx.x < MAXC) a.rr_part[t * MAXC + threadIdx.x] = outv[threadIdx.x];
  __syncthreads();
  block_reduce_cols<MAXC>(sr, sred, outv);
  if (threadIdx.x < MAXC) {
    a.SR_part[t * MAXC + threadIdx.x] = outv[threadIdx.x];
    a.SP0[t * MAXC + threadIdx.x] = outv[threadIdx.x];
  }
  if (!a.nofin && last_cta(&a.st->ticket[FIN_INIT])) {
    fin_init_body(a.st, a.prm, a.rr_part, a.L.n_tiles, ncol, NT / 32);
    if (threadIdx.x == 0) a.st->ticket[FIN_INIT] = 0;
  }
}

// ---------------------------------------------------------------------------------------
// Fused apply, persistent and warp-specialised.  CTA c owns clusters c, c+G, ... (tiles are
// whole clusters).  Warp NWC (the last) is the TMA producer; warps 0..NWC-1 consume.
// For cluster i:
//   D_i    = (fuse_p ? R + beta o P_old : D)      inputs TMA-staged by the producer
//   T_i    = mscale * sum_j Mp[i][j] S_j(D)       (low-rank, Eq. 19-21; all of this CTA's
//                                                   clusters computed once at kernel start)
//   BD     = B_i D_i: B_i (H or G, ld_i x ld_i column-major, contiguous) streams through an
//            nstage-deep shared-memory ring of KC-column chunks (1-D TMA bulk copies,
//            full/empty mbarriers per slot; no CTA-wide barrier in the stream)
//   val    = a D + b_i BD + u_i T_i                (Eq. 23-25 modes)
//   out    = cA val + cV D + cP P2                 (Q(A) / trace combines)
// Consumer mapping: thread -> (row quad rq, k-group g), g in the low lane bits (KG lanes per
// row quad, KG a power of two): each thread accumulates 4 rows x NCP columns over the chunk
// columns kk = g (mod KG); the KG partial sums are combined with xor shuffles.
// Epilogue: per-cluster partials of u^T out (next apply's S) or of out . Y2 (CG / trace dots).
constexpr int NTA = 256;              // threads per apply CTA (2 CTAs per SM)
constexpr int NWC = NTA / 32 - 1;     // consumer warps
constexpr int NTC = NWC * 32;         // consumer threads

__device__ __forceinline__ void cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(NTC) : "memory");
}

template <int NCP>
__device__ __forceinline__ void cons_reduce_cols(double (&v)[NCP], double* sred, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < NCP; ++c) v[c] = warp_sum(v[c]);
  cons_sync();
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < NCP; ++c) sred[wid * NCP + c] = v[c];
  }
  cons_sync();
  if (threadIdx.x < NCP) {
    double s = 0.0;
    for (int w = 0; w < NWC; ++w) s += sred[w * NCP + threadIdx.x];
    out[threadIdx.x] = s;
  }
  cons_sync();
}

template <int RPT>
__device__ __forceinline__ int apply_kg(int ld) {
  const int rq = ld / RPT;
  int kg = 1;
  while (kg < 8 && rq * kg * 2 <= NTC) kg <<= 1;
  return kg;
}
__device__ __forceinline__ int apply_kc(int ld, int slot, int kg) {
  int kc = max(1, slot / ld);
  if (kc >= kg) kc = (kc / kg) * kg;
  return kc;
}

template <int NCP>
__global__ void __launch_bounds__(NTA, 2) apply_kernel(ApplyArgs a) {
  constexpr int RPT = (NCP <= 10) ? 4 : 2;   // rows per consumer thread (register budget)
  if (a.gate && !a.st->any_active) return;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t empty[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t dbar, dfree;
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int n_c = a.L.n_c, n_tiles = a.L.n_tiles;
  const int64_t n_pad = a.L.n_pad;
  const int ncol = a.ncol;
  const EvalParams* P = a.prm;
  const int par = a.st->par;
  const double* B = P->B;
  const bool useB = (B != nullptr);
  const int slot = a.slot_doubles;
  const int nstage = a.nstage;
  const int G = gridDim.x;
  const int nmine = (n_tiles - static_cast<int>(blockIdx.x) + G - 1) / G;
  const int nsrc = a.fuse_p ? 2 : 1;
  double* ring = sm;                                         // nstage * slot (useB only)
  double* stg = ring + (useB ? nstage * slot : 0);           // 2 * ncol * ld_max (staged D inputs)
  double* Dsm = stg + 2 * ncol * a.ld_max;                   // ld_max * NCP (row-major Dsm[k*NCP+c])
  double* sred = Dsm + a.ld_max * NCP;                       // NWC * NCP
  double* Esm = sred + NWC * NCP;                            // NCP
  double* cb = Esm + NCP;                                    // NCP beta ; NCP active
  const double* Pold = a.fuse_p ? a.Pbuf[par] : nullptr;
  double* Pnew = a.fuse_p ? a.Pbuf[par ^ 1] : nullptr;
  const double* SPo = a.fuse_p ? a.SPbuf[par] : nullptr;
  const double* P2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.P2;
  const double* Y2 = a.use_par_p2 ? a.Pbuf[par ^ 1] : a.Y2;
  if (tid == 0) {
    for (int s_ = 0; s_ < nstage; ++s_) { mbar_init(&full[s_], 1); mbar_init(&empty[s_], NWC); }
    mbar_init(&dbar, 1);
    mbar_init(&dfree, 1);
    fence_mbar_init();
  }
  if (tid < NCP) {
    cb[tid] = (tid < ncol) ? a.st->beta[tid] : 0.0;
    cb[NCP + tid] = (tid < ncol) ? static_cast<double>(a.st->active[tid]) : 0.0;
  }
  __syncthreads();
  // TMA producer (lane 0 of warp NWC): work items in order: per tile q, the staged D inputs,
  // then the KC-column chunks of B_i.  prefill=true stops at the first item that would wait.
  int ct = blockIdx.x, cq = 0, ck0 = 0;
  bool cstaged = false;
  uint32_t pseq = 0;
  auto produce = [&](bool prefill) {
    while (ct < n_tiles) {
      const int i = a.L.tiles[ct].blk;
      const int ld = a.L.ld[i];
      if (!cstaged) {
        if (cq > 0) {
          if (prefill) return;
          mbar_wait(&dfree, static_cast<uint32_t>((cq - 1) & 1));
        }
        const int64_t p0 = a.L.poff[i];
        const uint32_t cbytes = static_cast<uint32_t>(ld) * 8u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&dbar, cbytes * ncol * nsrc);
        for (int c = 0; c < ncol; ++c) {
          tma_load_1d(stg + c * ld, a.D + c * n_pad + p0, cbytes, &dbar);
          if (nsrc == 2) tma_load_1d(stg + (ncol + c) * ld, Pold + c * n_pad + p0, cbytes, &dbar);
        }
        cstaged = true;
        ck0 = 0;
      }
      if (useB) {
        const int KC = apply_kc(ld, slot, apply_kg<RPT>(ld));
        const double* Bi = B + a.L.boff[i];
        while (ck0 < ld) {
          const int s_ = static_cast<int>(pseq % nstage);
          const uint32_t use = pseq / nstage;
          if (use > 0) {
            if (prefill) return;
            mbar_wait(&empty[s_], (use - 1) & 1u);
          }
          const int kc = min(KC, ld - ck0);
          const uint32_t bytes = static_cast<uint32_t>(kc) * ld * 8u;
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full[s_], bytes);
          tma_load_1d(ring + s_ * slot, Bi + static_cast<int64_t>(ck0) * ld, bytes, &full[s_]);
          ck0 += KC;
          ++pseq;
        }
      }
      ct += G;
      ++cq;
      cstaged = false;
    }
  };

  if (wid == NWC) {
    // ============================ producer warp ============================
    if (lane == 0) produce(false);
  } else {
    // ============================ consumer warps ============================
    uint32_t seq = 0;
    int q = 0;
    for (int t = blockIdx.x; t < n_tiles; t += G, ++q) {
      const TileDesc td = a.L.tiles[t];
      const int i = td.blk, ld = a.L.ld[i];
      const int64_t p0 = a.L.poff[i];
      // 1. D_i from the staged inputs (fused: D = R + beta o P_old, P_new written back)
      mbar_wait(&dbar, static_cast<uint32_t>(q & 1));
      for (int idx = tid; idx < ld * NCP; idx += NTC) {
        const int c = idx / ld, k = idx % ld;
        double v = 0.0;
        if (c < ncol) {
          v = stg[c * ld + k];
          if (a.fuse_p) {
            const double po = stg[(ncol + c) * ld + k];
            v = (cb[NCP + c] != 0.0) ? v + cb[c] * po : po;
            Pnew[c * n_pad + p0 + k] = v;
          }
        }
        Dsm[k * NCP + c] = v;
      }
      cons_sync();                                           // stg consumed, Dsm ready
      if (tid == 0) mbar_arrive(&dfree);
      // 2. block term from the TMA ring
      const int KG = apply_kg<RPT>(ld);
      const int RQ = ld / RPT;
      const int rq = tid / KG, g = tid % KG;
      const bool act = rq < RQ;
      const int r = RPT * rq;
      double acc[RPT][NCP];
#pragma unroll
      for (int h = 0; h < RPT; ++h)
#pragma unroll
        for (int c = 0; c < NCP; ++c) acc[h][c] = 0.0;
      if (useB) {
        const int KC = apply_kc(ld, slot, KG);
        for (int k0 = 0; k0 < ld; k0 += KC, ++seq) {
          const int kc = min(KC, ld - k0);
          const int s_ = static_cast<int>(seq % nstage);
          mbar_wait(&full[s_], (seq / nstage) & 1u);
          const double* cbuf = ring + s_ * slot;
          if (act && !(a.dbg & 1)) {
            for (int kk = g; kk < kc; kk += KG) {
              double bv[RPT];
#pragma unroll
              for (int h2 = 0; h2 < RPT / 2; ++h2) {
                const double2 b2 = *reinterpret_cast<const double2*>(cbuf + kk * ld + r + 2 * h2);
                bv[2 * h2] = b2.x;
                bv[2 * h2 + 1] = b2.y;
              }
              const double2* dk = reinterpret_cast<const double2*>(Dsm + (k0 + kk) * NCP);
#pragma unroll
              for (int c2 = 0; c2 < NCP / 2; ++c2) {
                const double2 dv = dk[c2];
#pragma unroll
                for (int h = 0; h < RPT; ++h) {
                  acc[h][2 * c2] = fma(bv[h], dv.x, acc[h][2 * c2]);
                  acc[h][2 * c2 + 1] = fma(bv[h], dv.y, acc[h][2 * c2 + 1]);
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s_]);
        }
        // combine the KG k-group partials (adjacent lanes) with xor shuffles
        for (int o = 1; o < KG; o <<= 1) {
#pragma unroll
          for (int h = 0; h < RPT; ++h)
#pragma unroll
            for (int c = 0; c < NCP; ++c) acc[h][c] += __shfl_xor_sync(0xffffffffu, acc[h][c], o);
        }
      }
      // 3. epilogue: after the xor all-reduce every k-group lane holds the row-quad sums;
      //    lane g writes the columns c with c % KG == g
      double ep[NCP];
#pragma unroll
      for (int c = 0; c < NCP; ++c) ep[c] = 0.0;
      if (act && !(a.dbg & 2)) {
        const double bi = P->b0 + P->b1 * a.jitter[i];
        const double pa = P->a, ms = P->mscale;
        const double* Tq = a.Tbuf + static_cast<int64_t>(i) * MAXC;
        double uu[RPT];
#pragma unroll
        for (int h = 0; h < RPT; ++h) uu[h] = a.u[p0 + r + h];
#pragma unroll
        for (int c = 0; c < NCP; ++c) {
          if (c < ncol && (c % KG) == g) {
            const int64_t gb = c * n_pad + p0 + r;
            double p2v[RPT], y2v[RPT];
#pragma unroll
            for (int h = 0; h < RPT; ++h) {
              p2v[h] = P2 ? P2[gb + h] : 0.0;
              y2v[h] = (a.epi == EPI_S) ? uu[h] : Y2[gb + h];
            }
#pragma unroll
            for (int h = 0; h < RPT; ++h) {
              const double d = Dsm[(r + h) * NCP + c];
              double val = pa * d;
              if (useB) val += bi * acc[h][c];
              val += uu[h] * (ms * Tq[c]);
              double o = a.cA[c] * val + a.cV[c] * d;
              if (P2) o += a.cP[c] * p2v[h];
              a.out[gb + h] = o;
              ep[c] += o * y2v[h];
            }
          }
        }
      }
      cons_reduce_cols<NCP>(ep, sred, Esm);
      if (tid < ncol) {
        if (a.epi == EPI_S) a.Sout[t * MAXC + tid] = Esm[tid];
        else a.dots[t * MAXC + tid] = Esm[tid];
      }
    }
  }
  // 4. finaliser (last CTA; one warp per column)
  if (a.fin != FIN_NONE) {
    if (last_cta(&a.st->ticket[a.fin])) {
      CGState* st = a.st;
      fin_alpha_trace_body(a.fin, st, a.dots, n_tiles, ncol, a.alpha_hist, a.hist_stride, NTA / 32);
      __syncthreads();
      if (tid == 0) st->ticket[a.fin] = 0;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Fused apply on the FP64 tensor pipe (DMMA mma.sync m8n8k4) for the paper's batch shape
// c = 1 + m = 9 columns (m = 8 probes).  Same contract as apply_kernel; the block
// product B_i D_i is split as
//   probe columns (8):  out_p[r, 0:8] += B_i[r, k:k+4] D_p[k:k+4, 0:8]   one m8n8k4 per 8 rows x 4 k
//   y column (1):       out_y[r]      += B_i[r, k] y_k                     one DFMA per A fragment
// so every issued FMA is useful (no column padding) and one DMMA replaces 8 DFMA instructions.
// Persistent CTAs (clusters c, c+G, ...), warp NWM (the last) drives the TMA ring of B_i chunks;
// the NWM consumer warps own the 8-row m-tiles mt = w, w + NWM, ... of the cluster and run over
// every chunk column.  D_i (and P_new = R + beta o P_old for the fused first apply) is read from
// L2/HBM once per cluster into shared memory: D_p as [k][LDP] with LDP = 12 (conflict-free
// B-fragment loads), y as [k].
constexpr int NWM = 7;                    // consumer warps of the DMMA apply (2 CTAs x 8 warps / SM)
constexpr int NTM = (NWM + 1) * 32;       // + 1 TMA producer warp
constexpr int LDP = 12;                   // row stride of the probe block in shared memory
constexpr int NW_SMALL = 3;               // consumer warps of the 4-CTA/SM DMMA apply (ld <= 9 * 3 * 8 = 216)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void mma_sync_consumers() {
  asm volatile("bar.sync 1, %0;" ::"r"(NWM * 32) : "memory");
}
template <int NW>
__device__ __forceinline__ void bar_consumers() {
  asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
}

// NW: consumer warps.  NW = NW (7): 2 CTAs per SM, persistent over clusters.  NW = 3 (128
// threads, <= 128 registers): 4 CTAs per SM, so that at C3 every cluster has its own CTA and the
// per-cluster phases (forming D_i, the epilogue) of co-resident CTAs overlap each other's streams.
template <int MTMAX, typename TB, int NW>   // m-tiles per warp; TB: stored element of B
__global__ void __launch_bounds__((NW + 1) * 32, (NW >= 7) ? 2 : 4) apply_mma_kernel(ApplyArgs a) {
  constexpr int EG = 2;                      // m-tiles per epilogue load group
  constexpr int NCPE = 10;                 // epilogue column slots (9 used)
  if (a.gate && !a.st->any_active) return;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t empty[MAX_NSTAGE];
  __shared__ double sred[NW * NCPE];
  __shared__ double Esm[NCPE];
  __shared__ double cb[2 * NCPE];
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int n_tiles = a.L.n_tiles;
  const int64_t n_pad = a.L.n_pad;
  const int ncol = a.ncol;                 // == 9
  const EvalParams* P = a.prm;
  const int par = a.st->par;
  const TB* B = (sizeof(TB) == 4) ? reinterpret_cast<const TB*>(P->B32) : reinterpret_cast<const TB*>(P->B);
  const bool useB = (P->B != nullptr);
  constexpr int EPS = 8 / static_cast<int>(sizeof(TB));   // B elements per 8-byte slot unit
  const int slot = a.slot_doubles;
  const int nstage = a.nstage;
  const int G = gridDim.x;
  // progressive D (dstride > 0, with a block term): the TMA producer also brings each chunk's k-rows
  // of D (and of P_old for the fused first apply) into a per-stage area next to the B chunk, so the
  // consumers start on the block stream at once instead of first loading all of D_i
  const int pd = a.dstride;
  const bool prog = useB && pd > 0;
  double* ring = sm;                                         // nstage * slot (useB only)
  double* Dst = ring + (useB ? nstage * slot : 0);           // prog: nstage * 18 * pd ([c][pd], R then P_old)
  double* Dp = Dst + (prog ? nstage * 18 * pd : 0);          // ld_max * LDP
  double* ys = Dp + a.ld_max * LDP;                          // ld_max
  // dbuf: a second D_i buffer.  An apply whose D is a plain vector (not the fused R + beta P_old)
  // copies the NEXT cluster's D_i into it with cp.async while this cluster streams, so only a
  // CTA's first cluster waits for its D_i
  double* Dp1 = ys + a.ld_max;                               // dbuf: ld_max * LDP
  double* ys1 = Dp1 + a.ld_max * LDP;                        // dbuf: ld_max
  double* Pst = ys1 + a.ld_max;                              // dbuf == 2: next cluster's P_old [9][ld]
  // (dbuf == 2: the fused apply also prefetches R and P_old and forms R + beta o P_old at the start)
  const bool dpre = a.dbuf && (!a.fuse_p || a.dbuf == 2) && !prog && !(a.dbg & 64);
  bool have_next = false;                                    // D_i of this cluster already copied
  const double* Pold = a.fuse_p ? a.Pbuf[par] : nullptr;
  double* Pnew = a.fuse_p ? a.Pbuf[par ^ 1] : nullptr;
  const double* P2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.P2;
  const double* Y2 = a.use_par_p2 ? a.Pbuf[par ^ 1] : a.Y2;
  if (tid == 0) {
    for (int s_ = 0; s_ < nstage; ++s_) { mbar_init(&full[s_], 1); mbar_init(&empty[s_], NW); }
    fence_mbar_init();
  }
  if (tid < NCPE) {
    cb[tid] = (tid < ncol) ? a.st->beta[tid] : 0.0;
    cb[NCPE + tid] = (tid < ncol) ? static_cast<double>(a.st->active[tid]) : 0.0;
  }
  __syncthreads();
  if (wid == NW) {
    // ============================ TMA producer ============================
    if (lane == 0 && useB) {
      uint32_t pseq = 0;
      // cluster descriptors are loaded one cluster ahead, and the L2 prefetches are issued after the
      // cluster's first chunk, so no chain of dependent descriptor loads sits between the last chunk
      // of one cluster and the first chunk of the next (it drained the ring at every transition)
      int i_nx = 0, ld_nx = 0;
      int64_t bo_nx = 0, p0_nx = 0;
      if (static_cast<int>(blockIdx.x) < n_tiles) {
        i_nx = a.L.tiles[blockIdx.x].blk;
        ld_nx = a.L.ld[i_nx];
        bo_nx = a.L.boff[i_nx];
        p0_nx = a.L.poff[i_nx];
      }
      for (int t = blockIdx.x; t < n_tiles; t += G) {
        const int i = i_nx, ld = ld_nx;
        const int64_t p0 = p0_nx;
        const TB* Bi = B + bo_nx;
        const int tn = t + G;
        if (tn < n_tiles) {
          i_nx = a.L.tiles[tn].blk;
          ld_nx = a.L.ld[i_nx];
          bo_nx = a.L.boff[i_nx];
          p0_nx = a.L.poff[i_nx];
        }
        const int KC = max(4, (EPS * slot / ld) & ~3);
        for (int ck0 = 0; ck0 < ld; ck0 += KC, ++pseq) {
          const int s_ = static_cast<int>(pseq % nstage);
          const uint32_t use = pseq / nstage;
          if (use > 0) mbar_wait(&empty[s_], (use - 1) & 1u);
          const int kc = min(KC, ld - ck0);
          const uint32_t bytes = static_cast<uint32_t>(kc) * ld * static_cast<uint32_t>(sizeof(TB));
          const uint32_t dseg = static_cast<uint32_t>(kc) * 8u;
          const uint32_t dbytes = prog ? dseg * 9u * (a.fuse_p ? 2u : 1u) : 0u;
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full[s_], bytes + dbytes);
          tma_load_1d(ring + s_ * slot, Bi + static_cast<int64_t>(ck0) * ld, bytes, &full[s_]);
          if (prog) {
            double* ds = Dst + s_ * 18 * pd;
            for (int c = 0; c < 9; ++c) {
              tma_load_1d(ds + c * pd, a.D + c * n_pad + p0 + ck0, dseg, &full[s_]);
              if (a.fuse_p) tma_load_1d(ds + (9 + c) * pd, Pold + c * n_pad + p0 + ck0, dseg, &full[s_]);
            }
          }
          if (ck0 == 0 && !(a.dbg & 32)) {
            // warm L2 with this cluster's epilogue inputs and the next cluster's D inputs, so the
            // consumers' plain loads there do not queue behind the B stream in DRAM
            const uint32_t cb8 = static_cast<uint32_t>(ld) * 8u;
            tma_prefetch_l2(a.u + p0, cb8);
            for (int c = 0; c < ncol; ++c) {
              if (P2) tma_prefetch_l2(P2 + c * n_pad + p0, cb8);
              if (a.epi != EPI_S && Y2 != P2 && a.use_par_p2 != 2) tma_prefetch_l2(Y2 + c * n_pad + p0, cb8);
            }
            if (tn < n_tiles) {
              const uint32_t cbn = static_cast<uint32_t>(ld_nx) * 8u;
              for (int c = 0; c < ncol; ++c) {
                tma_prefetch_l2(a.D + c * n_pad + p0_nx, cbn);
                if (a.fuse_p) tma_prefetch_l2(Pold + c * n_pad + p0_nx, cbn);
              }
            }
          }
        }
      }
    }
    return;
  }
  // ============================ consumers ============================
  const int qr = lane >> 2, qc = lane & 3;   // fragment row / k (A), k / n (B) coordinates
  uint32_t seq = 0;
  // (a.dbg & 16: per-CTA phase timestamps via printf, timing experiments only)
  unsigned long long tsm[1 + 3 * 16];
  int nts = 0;
  auto stamp = [&]() {
    if ((a.dbg & 16) && tid == 0 && nts < 1 + 3 * 16) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tsm[nts++] = tt;
    }
  };
  stamp();
  // cluster descriptors one cluster ahead (their dependent loads overlap the previous cluster)
  int ci_nx = 0, cld_nx = 0;
  int64_t cp0_nx = 0;
  if (static_cast<int>(blockIdx.x) < n_tiles) {
    ci_nx = a.L.tiles[blockIdx.x].blk;
    cld_nx = a.L.ld[ci_nx];
    cp0_nx = a.L.poff[ci_nx];
  }
  for (int t = blockIdx.x; t < n_tiles; t += G) {
    const int i = ci_nx, ld = cld_nx;
    const int64_t p0 = cp0_nx;
    if (t + G < n_tiles) {
      ci_nx = a.L.tiles[t + G].blk;
      cld_nx = a.L.ld[ci_nx];
      cp0_nx = a.L.poff[ci_nx];
    }
    const int mtt = ld >> 3;                               // m-tiles of the cluster
    // 1. D_i -> shared (fused: D = R + beta o P_old for active columns, P_new written back);
    //    loads batched 4 deep per thread so one cluster costs ~one memory round trip
    if (prog) {
      // (D_i arrives chunk by chunk with the block stream)
    } else if (have_next) {
      cp_async_wait_all();                                   // (made visible by the barrier below)
      if (a.fuse_p) {
        bar_consumers<NW>();
        for (int idx = tid; idx < ld * 9; idx += NW * 32) {
          const int c = idx / ld, k = idx - c * ld;
          double* dst = (c == 0) ? ys + k : Dp + k * LDP + (c - 1);
          const double po = Pst[c * ld + k];
          const double x = (cb[NCPE + c] != 0.0) ? *dst + cb[c] * po : po;
          Pnew[c * n_pad + p0 + k] = x;
          *dst = x;
        }
      }
    } else if (a.dbg & 64) {
      // timing experiment only: no D_i load (results invalid)
    } else if (a.dbg & 4) {
      for (int idx = tid; idx < ld * 9; idx += NW * 32) {
        const int c = idx / ld, k = idx - c * ld;
        const int64_t gi = c * n_pad + p0 + k;
        double v = a.D[gi];
        if (a.fuse_p) {
          const double po = Pold[gi];
          v = (cb[NCPE + c] != 0.0) ? v + cb[c] * po : po;
          Pnew[gi] = v;
        }
        if (c == 0) ys[k] = v; else Dp[k * LDP + (c - 1)] = v;
      }
    } else {
      /* batched conversion below */
      const int tot = ld * 9;
      constexpr int CU = (NW < 5) ? 8 : 4;
      for (int base = 0; base < tot; base += CU * NW * 32) {
        double v[CU], po[CU];
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int idx = base + u * NW * 32 + tid;
          v[u] = 0.0; po[u] = 0.0;
          if (idx < tot) {
            const int c = idx / ld, k = idx - c * ld;
            const int64_t gi = c * n_pad + p0 + k;
            v[u] = __ldg(a.D + gi);
            if (a.fuse_p) po[u] = __ldg(Pold + gi);
          }
        }
#pragma unroll
        for (int u = 0; u < CU; ++u) {
          const int idx = base + u * NW * 32 + tid;
          if (idx < tot) {
            const int c = idx / ld, k = idx - c * ld;
            double x = v[u];
            if (a.fuse_p) {
              x = (cb[NCPE + c] != 0.0) ? x + cb[c] * po[u] : po[u];
              Pnew[c * n_pad + p0 + k] = x;
            }
            if (c == 0) ys[k] = x; else Dp[k * LDP + (c - 1)] = x;
          }
        }
      }
    }
    bar_consumers<NW>();
    have_next = false;
    if (dpre && t + G < n_tiles) {
      // the next cluster's D_i -> the other buffer, asynchronously (waited for at its start)
      const int ldn = cld_nx;
      const int64_t pn = cp0_nx;
      for (int idx = tid; idx < ldn * 9; idx += NW * 32) {
        const int c = idx / ldn, k = idx - c * ldn;
        const double* src = a.D + c * n_pad + pn + k;
        cp_async8((c == 0) ? ys1 + k : Dp1 + k * LDP + (c - 1), src);
        if (a.fuse_p) cp_async8(Pst + c * ldn + k, Pold + c * n_pad + pn + k);
      }
      cp_async_commit();
      have_next = true;
    }
    stamp();
    // 2. block term: DMMA over the ring chunks
    double acc0[MTMAX], acc1[MTMAX], accy[MTMAX];
#pragma unroll
    for (int j = 0; j < MTMAX; ++j) { acc0[j] = 0.0; acc1[j] = 0.0; accy[j] = 0.0; }
    if (useB) {
      const int KC = max(4, (EPS * slot / ld) & ~3);
      for (int k0 = 0; k0 < ld; k0 += KC, ++seq) {
        const int kc = min(KC, ld - k0);
        const int s_ = static_cast<int>(seq % nstage);
        mbar_wait(&full[s_], (seq / nstage) & 1u);
        const TB* cbuf = reinterpret_cast<const TB*>(ring + s_ * slot);
        if (prog) {
          const double* ds = Dst + s_ * 18 * pd;
          // the D value of column c at chunk row kk (fused: R + beta o P_old for active columns)
          auto dval = [&](int c, int kk) -> double {
            double v = ds[c * pd + kk];
            if (a.fuse_p) {
              const double po = ds[(9 + c) * pd + kk];
              v = (cb[NCPE + c] != 0.0) ? v + cb[c] * po : po;
            }
            return v;
          };
          for (int kq = 0; kq < kc; kq += 4) {
            const int kk = kq + qc;
            const double bfr = dval(1 + qr, kk);             // B fragment: D_p[k][n = qr]
            const double yv = dval(0, kk);
            const TB* acol = cbuf + kk * ld + qr;            // A fragment base: B_i[r][k]
#pragma unroll
            for (int j = 0; j < MTMAX; ++j) {
              const int mt = wid + j * NW;
              if (mt < mtt) {
                const double afr = static_cast<double>(acol[mt * 8]);
                dmma884(acc0[j], acc1[j], afr, bfr);
                accy[j] = fma(afr, yv, accy[j]);
              }
            }
          }
          // one warp per chunk keeps D_i for the epilogue (and writes P_new of the fused apply)
          if (wid == static_cast<int>(seq % NW)) {
            for (int idx = lane; idx < 9 * kc; idx += 32) {
              const int c = idx / kc, kk = idx - c * kc;
              const double v = dval(c, kk);
              if (a.fuse_p) Pnew[c * n_pad + p0 + k0 + kk] = v;
              if (c == 0) ys[k0 + kk] = v; else Dp[(k0 + kk) * LDP + (c - 1)] = v;
            }
          }
        } else if (!(a.dbg & 1)) {
          for (int kq = 0; kq < kc; kq += 4) {
            const int k = k0 + kq + qc;                      // this lane's k in the cluster
            const double bfr = Dp[k * LDP + qr];             // B fragment: D_p[k][n = qr]
            const double yv = ys[k];
            const TB* acol = cbuf + (kq + qc) * ld + qr;     // A fragment base: B_i[r][k]
#pragma unroll
            for (int j = 0; j < MTMAX; ++j) {
              const int mt = wid + j * NW;
              if (mt < mtt) {
                const double afr = static_cast<double>(acol[mt * 8]);
                dmma884(acc0[j], acc1[j], afr, bfr);
                accy[j] = fma(afr, yv, accy[j]);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s_]);
      }
    }
    if (prog) bar_consumers<NW>();            // D_i complete in shared memory for the epilogue
    stamp();
    // y column: reduce the 4 k-lanes of each row quad
#pragma unroll
    for (int j = 0; j < MTMAX; ++j) {
      accy[j] += __shfl_xor_sync(0xffffffffu, accy[j], 1);
      accy[j] += __shfl_xor_sync(0xffffffffu, accy[j], 2);
    }
    // 3. epilogue: lane owns row r = 8 mt + qr, probe columns c = 1 + 2 qc + {0, 1}, and the y
    //    column when qc == 0
    double ep[NCPE];
#pragma unroll
    for (int c = 0; c < NCPE; ++c) ep[c] = 0.0;
    if (!(a.dbg & 2)) {
      const double bi = P->b0 + P->b1 * a.jitter[i];
      const double pa = P->a, ms = P->mscale;
      const double* Tq = a.Tbuf + static_cast<int64_t>(i) * MAXC;
      const int c0 = 1 + 2 * qc;
#pragma unroll
      for (int jg = 0; jg < MTMAX; jg += EG) {
        // load phase (all global reads of EG m-tiles in flight together), then compute
        double uu[EG], p2v[EG][3], y2v[EG][3];
#pragma unroll
        for (int jj = 0; jj < EG; ++jj) {
          const int mt = wid + (jg + jj) * NW;
          const bool on = mt < mtt;
          const int r = mt * 8 + qr;
          uu[jj] = on ? __ldg(a.u + p0 + r) : 0.0;
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            const int c = (e < 2) ? c0 + e : 0;
            const int64_t gi = c * n_pad + p0 + r;
            const bool le = on && (e < 2 || qc == 0);
            p2v[jj][e] = (le && P2) ? P2[gi] : 0.0;
            // (the Q(A) apply's dot partner is its combine term P_new: one load serves both)
            y2v[jj][e] = (le && a.epi != EPI_S && a.use_par_p2 != 2) ? ((Y2 == P2) ? p2v[jj][e] : Y2[gi]) : 0.0;
          }
        }
#pragma unroll
        for (int jj = 0; jj < EG; ++jj) {
          const int j = jg + jj;
          const int mt = wid + j * NW;
          if (mt < mtt) {
            const int r = mt * 8 + qr;
#pragma unroll
            for (int e = 0; e < 3; ++e) {
              if (e == 2 && qc != 0) continue;
              const int c = (e < 2) ? c0 + e : 0;
              const double bd = (e == 0) ? acc0[j] : (e == 1) ? acc1[j] : accy[j];
              const double d = (e < 2) ? Dp[r * LDP + c - 1] : ys[r];
              const int64_t gi = c * n_pad + p0 + r;
              double val = pa * d;
              if (useB) val += bi * bd;
              val += uu[jj] * (ms * Tq[c]);
              double o = a.cA[c] * val + a.cV[c] * d;
              if (P2) o += a.cP[c] * p2v[jj][e];
              a.out[gi] = o;
              // (mBCG: the dot partner is P_new = D_i itself, already in shared memory)
              const double y2 = (a.epi == EPI_S) ? uu[jj] : (a.use_par_p2 == 2) ? d : y2v[jj][e];
              // ep[c] += o * y2 with a compile-time column index
#pragma unroll
              for (int cc = 0; cc < 9; ++cc)
                if (cc == c) ep[cc] += o * y2;
            }
          }
        }
      }
    }
    // CTA-wide fixed-order column sums of ep over the consumer warps
#pragma unroll
    for (int c = 0; c < NCPE; ++c) ep[c] = warp_sum(ep[c]);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < NCPE; ++c) sred[wid * NCPE + c] = ep[c];
    }
    bar_consumers<NW>();
    if (tid < ncol) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += sred[w * NCPE + tid];
      if (a.epi == EPI_S) a.Sout[t * MAXC + tid] = s;
      else a.dots[t * MAXC + tid] = s;
    }
    bar_consumers<NW>();                                   // sred / Dp / ys reuse
    if (dpre) {                                            // the prefetched buffer becomes current
      double* tp = Dp; Dp = Dp1; Dp1 = tp;
      tp = ys; ys = ys1; ys1 = tp;
    }
    stamp();
  }
  if ((a.dbg & 16) && tid == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    for (int k = 0; k < nts; ++k)
      printf("T %d %u %d %llu\n", blockIdx.x, smid, k, tsm[k]);
  }
  // 4. finaliser (last CTA among the consumers; one warp per column)
  if (a.fin != FIN_NONE) {
    __shared__ int s_last;
    __threadfence();
    bar_consumers<NW>();
    if (tid == 0) {
      const unsigned int tk = atomicAdd(&a.st->ticket[a.fin], 1u);
      s_last = (tk == gridDim.x - 1);
    }
    bar_consumers<NW>();
    if (s_last) {
      __threadfence();
      CGState* st = a.st;
      fin_alpha_trace_body(a.fin, st, a.dots, n_tiles, ncol, a.alpha_hist, a.hist_stride, NW);
      bar_consumers<NW>();
      if (tid == 0) st->ticket[a.fin] = 0;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Cross-perturbation batched apply (NEXT-3): NG evaluations whose operators share
// the block term B (the noise- and scale-steps all use H, Eq. 24-25) run their CG in lockstep and
// their applies are ONE launch that streams each B_i once for all of them.  Group g has its own
// ApplyArgs (EvalParams, CG state, vectors, partials); the kernel is apply_mma_kernel with the
// probe block of group g in n-tile g and its y column as a DFMA on the same A fragment.
constexpr int MGMAX = 4;
struct MultiApplyArgs {
  ApplyArgs g[MGMAX];
  int ng;
};

template <int MTMAX, int NG>
__global__ void __launch_bounds__(NTM, 2) apply_multi_kernel(const __grid_constant__ MultiApplyArgs ma) {
  constexpr int NCPE = 10;
  constexpr int LDG = (NG == 1) ? 12 : (NG == 2) ? 20 : 36;   // probe row stride: 8*NG (+pad), = 4 (mod 16)
  const ApplyArgs& a0 = ma.g[0];
  bool any = false;
#pragma unroll
  for (int g = 0; g < NG; ++g) any |= (!ma.g[g].gate || ma.g[g].st->any_active);
  if (!any) return;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t empty[MAX_NSTAGE];
  __shared__ double sred[NWM * NCPE];
  __shared__ double cb[NG][2 * NCPE];
  __shared__ int s_par[NG];
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int n_tiles = a0.L.n_tiles;
  const int64_t n_pad = a0.L.n_pad;
  const double* B = a0.prm->B;                 // shared by every group
  const bool useB = (B != nullptr);
  const int slot = a0.slot_doubles;
  const int nstage = a0.nstage;
  const int G = gridDim.x;
  double* ring = sm;
  double* Dp = ring + (useB ? nstage * slot : 0);          // ld_max * LDG: probes of group g at 8g
  double* ys = Dp + a0.ld_max * LDG;                       // NG * ld_max
  if (tid == 0) {
    for (int s_ = 0; s_ < nstage; ++s_) { mbar_init(&full[s_], 1); mbar_init(&empty[s_], NWM); }
    fence_mbar_init();
  }
  if (tid < NG) s_par[tid] = ma.g[tid].st->par;
  for (int t = tid; t < NG * NCPE; t += NTM) {
    const int g = t / NCPE, c = t % NCPE;
    const CGState* st = ma.g[g].st;
    cb[g][c] = (c < 9) ? st->beta[c] : 0.0;
    cb[g][NCPE + c] = (c < 9) ? static_cast<double>(st->active[c]) : 0.0;
  }
  __syncthreads();
  if (wid == NWM) {
    if (lane == 0 && useB) {
      uint32_t pseq = 0;
      for (int t = blockIdx.x; t < n_tiles; t += G) {
        const int i = a0.L.tiles[t].blk;
        const int ld = a0.L.ld[i];
        const int KC = max(4, (slot / ld) & ~3);
        const double* Bi = B + a0.L.boff[i];
        for (int ck0 = 0; ck0 < ld; ck0 += KC, ++pseq) {
          const int s_ = static_cast<int>(pseq % nstage);
          const uint32_t use = pseq / nstage;
          if (use > 0) mbar_wait(&empty[s_], (use - 1) & 1u);
          const int kc = min(KC, ld - ck0);
          const uint32_t bytes = static_cast<uint32_t>(kc) * ld * 8u;
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full[s_], bytes);
          tma_load_1d(ring + s_ * slot, Bi + static_cast<int64_t>(ck0) * ld, bytes, &full[s_]);
        }
      }
    }
    return;
  }
  const int qr = lane >> 2, qc = lane & 3;
  uint32_t seq = 0;
  for (int t = blockIdx.x; t < n_tiles; t += G) {
    const TileDesc td = a0.L.tiles[t];
    const int i = td.blk, ld = a0.L.ld[i];
    const int64_t p0 = a0.L.poff[i];
    const int mtt = ld >> 3;
    // 1. D_i of every group -> shared
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const ApplyArgs& a = ma.g[g];
      const int par = s_par[g];
      const double* Pold = a.fuse_p ? a.Pbuf[par] : nullptr;
      double* Pnew = a.fuse_p ? a.Pbuf[par ^ 1] : nullptr;
      for (int idx = tid; idx < ld * 9; idx += NWM * 32) {
        const int c = idx / ld, k = idx - c * ld;
        const int64_t gi = c * n_pad + p0 + k;
        double v = a.D[gi];
        if (a.fuse_p) {
          const double po = Pold[gi];
          v = (cb[g][NCPE + c] != 0.0) ? v + cb[g][c] * po : po;
          Pnew[gi] = v;
        }
        if (c == 0) ys[g * a0.ld_max + k] = v; else Dp[k * LDG + 8 * g + (c - 1)] = v;
      }
    }
    mma_sync_consumers();
    // 2. block term: one pass over B_i's chunks for all groups
    double acc0[MTMAX][NG], acc1[MTMAX][NG], accy[MTMAX][NG];
#pragma unroll
    for (int j = 0; j < MTMAX; ++j)
#pragma unroll
      for (int g = 0; g < NG; ++g) { acc0[j][g] = 0.0; acc1[j][g] = 0.0; accy[j][g] = 0.0; }
    if (useB) {
      const int KC = max(4, (slot / ld) & ~3);
      for (int k0 = 0; k0 < ld; k0 += KC, ++seq) {
        const int kc = min(KC, ld - k0);
        const int s_ = static_cast<int>(seq % nstage);
        mbar_wait(&full[s_], (seq / nstage) & 1u);
        const double* cbuf = ring + s_ * slot;
        for (int kq = 0; kq < kc; kq += 4) {
          const int k = k0 + kq + qc;
          double bfr[NG], yv[NG];
#pragma unroll
          for (int g = 0; g < NG; ++g) { bfr[g] = Dp[k * LDG + 8 * g + qr]; yv[g] = ys[g * a0.ld_max + k]; }
          const double* acol = cbuf + (kq + qc) * ld + qr;
#pragma unroll
          for (int j = 0; j < MTMAX; ++j) {
            const int mt = wid + j * NWM;
            if (mt < mtt) {
              const double afr = acol[mt * 8];
#pragma unroll
              for (int g = 0; g < NG; ++g) {
                dmma884(acc0[j][g], acc1[j][g], afr, bfr[g]);
                accy[j][g] = fma(afr, yv[g], accy[j][g]);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s_]);
      }
    }
#pragma unroll
    for (int j = 0; j < MTMAX; ++j)
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        accy[j][g] += __shfl_xor_sync(0xffffffffu, accy[j][g], 1);
        accy[j][g] += __shfl_xor_sync(0xffffffffu, accy[j][g], 2);
      }
    // 3. epilogue per group
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const ApplyArgs& a = ma.g[g];
      const EvalParams* P = a.prm;
      const int par = s_par[g];
      const double* P2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.P2;
      const double* Y2 = a.use_par_p2 ? a.Pbuf[par ^ 1] : a.Y2;
      double ep[NCPE];
#pragma unroll
      for (int c = 0; c < NCPE; ++c) ep[c] = 0.0;
      const bool gon = !a.gate || a.st->any_active;
      if (gon) {
        const double bi = P->b0 + P->b1 * a.jitter[i];
        const double pa = P->a, ms = P->mscale;
        const double* Tq = a.Tbuf + static_cast<int64_t>(i) * MAXC;
#pragma unroll
        for (int j = 0; j < MTMAX; ++j) {
          const int mt = wid + j * NWM;
          if (mt < mtt) {
            const int r = mt * 8 + qr;
            const double uu = a.u[p0 + r];
#pragma unroll
            for (int e = 0; e < 3; ++e) {
              if (e == 2 && qc != 0) continue;
              const int c = (e < 2) ? 1 + 2 * qc + e : 0;
              const double bd = (e == 0) ? acc0[j][g] : (e == 1) ? acc1[j][g] : accy[j][g];
              const double d = (e < 2) ? Dp[r * LDG + 8 * g + c - 1] : ys[g * a0.ld_max + r];
              const int64_t gi = c * n_pad + p0 + r;
              double val = pa * d;
              if (useB) val += bi * bd;
              val += uu * (ms * Tq[c]);
              double o = a.cA[c] * val + a.cV[c] * d;
              if (P2) o += a.cP[c] * P2[gi];
              a.out[gi] = o;
              const double y2 = (a.epi == EPI_S) ? uu : Y2[gi];
#pragma unroll
              for (int cc = 0; cc < 9; ++cc)
                if (cc == c) ep[cc] += o * y2;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NCPE; ++c) ep[c] = warp_sum(ep[c]);
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < NCPE; ++c) sred[wid * NCPE + c] = ep[c];
      }
      mma_sync_consumers();
      if (tid < 9) {
        double s = 0.0;
        for (int w = 0; w < NWM; ++w) s += sred[w * NCPE + tid];
        if (a.epi == EPI_S) a.Sout[t * MAXC + tid] = s;
        else a.dots[t * MAXC + tid] = s;
      }
      mma_sync_consumers();
    }
  }
  // 4. finalisers (last CTA; one warp per (group, column))
  if (a0.fin != FIN_NONE) {
    __shared__ int s_last;
    __threadfence();
    mma_sync_consumers();
    if (tid == 0) {
      const unsigned int tk = atomicAdd(&a0.st->ticket[a0.fin], 1u);
      s_last = (tk == gridDim.x - 1);
    }
    mma_sync_consumers();
    if (s_last) {
      __threadfence();
      for (int gc = wid; gc < NG * 9; gc += NWM) {
        const int g = gc / 9, c = gc % 9;
        const ApplyArgs& a = ma.g[g];
        CGState* st = a.st;
        if (a.gate && !st->any_active) continue;
        const double tot = col_total(a.dots, n_tiles, c);
        if (lane == 0) {
          if (a.fin == FIN_ALPHA) {
            if (st->active[c]) {
              const double al = st->rr[c] / tot;
              st->alpha[c] = al;
              a.alpha_hist[c * a.hist_stride + st->iters[c]] = al;
            }
          } else {
            if (c == 0) st->quad = tot; else st->t[c] = tot;
          }
        }
      }
      mma_sync_consumers();
      if (tid == 0) a0.st->ticket[a0.fin] = 0;
    }
  }
}

// Loop condition of a batched CG graph: continue while any group has an active column.
__global__ void cond_any_kernel(const CGState* s0, const CGState* s1, const CGState* s2, const CGState* s3,
                                int ng, unsigned long long cond) {
  int any = s0->any_active;
  if (ng > 1) any |= s1->any_active;
  if (ng > 2) any |= s2->any_active;
  if (ng > 3) any |= s3->any_active;
  cudaGraphSetConditional(cond, any ? 1u : 0u);
}

// ---------------------------------------------------------------------------------------
// Staged variant of the DMMA apply (1 CTA per SM): every per-cluster input is TMA-staged into
// shared memory by the producer warp ahead of use, so the consumers' cluster prologue (forming
// D_i) and epilogue run from shared memory instead of paying global-memory round trips that
// queue behind the B stream.  Producer work per owned cluster q (polled, non-blocking):
//   D(q): the 9 columns of D_i (+ the 9 of P_old when fused) -> stgD, after the consumers
//         released stgD from cluster q-1 (dfree);
//   E(q): u_i, the P2 and Y2 columns and the low-rank row T_i -> stgE, after the epilogue of
//         cluster q-1 released stgE (efree);
//   B(q): the KC-column chunks of B_i through the ring (full/empty barriers).
// Tile metadata of the CTA's clusters is loaded once into shared memory.
constexpr int MAXQ = 32;                  // clusters per CTA held in the metadata cache

template <int MTMAX>
__global__ void __launch_bounds__(NTM, 2) apply_mma_staged_kernel(ApplyArgs a) {
  constexpr int NCPE = 10;
  if (a.gate && !a.st->any_active) return;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t empty[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t dbar, dfree, ebar, efree;
  __shared__ double sred[NWM * NCPE];
  __shared__ double cb[2 * NCPE];
  __shared__ int q_ld[MAXQ];
  __shared__ int64_t q_p0[MAXQ], q_boff[MAXQ];
  __shared__ double q_bi[MAXQ];
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int n_tiles = a.L.n_tiles;
  const int64_t n_pad = a.L.n_pad;
  const int ncol = a.ncol;                 // == 9
  const EvalParams* P = a.prm;
  const int par = a.st->par;
  const double* B = P->B;
  const bool useB = (B != nullptr);
  const int slot = a.slot_doubles;
  const int nstage = a.nstage;
  const int G = gridDim.x;
  const int ldm = a.ld_max;
  const int nmine = (n_tiles - static_cast<int>(blockIdx.x) + G - 1) / G;
  const double* Pold = a.fuse_p ? a.Pbuf[par] : nullptr;
  double* Pnew = a.fuse_p ? a.Pbuf[par ^ 1] : nullptr;
  const double* P2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.P2;
  const double* Y2 = a.use_par_p2 ? a.Pbuf[par ^ 1] : a.Y2;
  const bool eY2 = (a.epi != EPI_S) && (Y2 != P2);          // Y2 needs its own staging
  double* ring = sm;                                         // nstage * slot
  double* stgD = ring + (useB ? nstage * slot : 0);          // 18 * ldm
  double* stgE = stgD + 18 * ldm;                            // u | P2 (9) | Y2 (9) | T (16)
  double* sT = stgE + 19 * ldm;
  double* Dp = sT + 16;                                      // ldm * LDP
  double* ys = Dp + ldm * LDP;                               // ldm
  if (tid == 0) {
    for (int s_ = 0; s_ < nstage; ++s_) { mbar_init(&full[s_], 1); mbar_init(&empty[s_], NWM); }
    mbar_init(&dbar, 1); mbar_init(&dfree, 1); mbar_init(&ebar, 1); mbar_init(&efree, 1);
    fence_mbar_init();
  }
  if (tid < NCPE) {
    cb[tid] = (tid < ncol) ? a.st->beta[tid] : 0.0;
    cb[NCPE + tid] = (tid < ncol) ? static_cast<double>(a.st->active[tid]) : 0.0;
  }
  for (int q = tid; q < nmine; q += NTM) {
    const int i = a.L.tiles[blockIdx.x + q * G].blk;
    q_ld[q] = a.L.ld[i];
    q_p0[q] = a.L.poff[i];
    q_boff[q] = a.L.boff[i];
    q_bi[q] = P->b0 + P->b1 * a.jitter[i];
  }
  __syncthreads();
  if (wid == NWM) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      int qD = 0, qE = 0, qB = 0, ck0 = 0;
      uint32_t pseq = 0;
      while (qD < nmine || qE < nmine || qB < nmine) {
        if (qD < nmine && qD <= qB + 1 && (qD == 0 || mbar_try_wait(&dfree, (qD - 1) & 1))) {
          const int ld = q_ld[qD];
          const int64_t p0 = q_p0[qD];
          const uint32_t cb8 = static_cast<uint32_t>(ld) * 8u;
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&dbar, cb8 * ncol * (a.fuse_p ? 2 : 1));
          for (int c = 0; c < ncol; ++c) {
            tma_load_1d(stgD + c * ld, a.D + c * n_pad + p0, cb8, &dbar);
            if (a.fuse_p) tma_load_1d(stgD + (9 + c) * ld, Pold + c * n_pad + p0, cb8, &dbar);
          }
          ++qD;
        }
        if (qE < nmine && qE <= qB && (qE == 0 || mbar_try_wait(&efree, (qE - 1) & 1))) {
          const int ld = q_ld[qE];
          const int64_t p0 = q_p0[qE];
          const int i = a.L.tiles[blockIdx.x + qE * G].blk;
          const uint32_t cb8 = static_cast<uint32_t>(ld) * 8u;
          const uint32_t tot = cb8 * (1 + (P2 ? ncol : 0) + (eY2 ? ncol : 0)) + 16u * 8u;
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&ebar, tot);
          tma_load_1d(stgE, a.u + p0, cb8, &ebar);
          for (int c = 0; c < ncol; ++c) {
            if (P2) tma_load_1d(stgE + (1 + c) * ld, P2 + c * n_pad + p0, cb8, &ebar);
            if (eY2) tma_load_1d(stgE + (10 + c) * ld, Y2 + c * n_pad + p0, cb8, &ebar);
          }
          tma_load_1d(sT, a.Tbuf + static_cast<int64_t>(i) * MAXC, 16u * 8u, &ebar);
          ++qE;
        }
        if (qB < nmine && qB < qD) {
          if (!useB) {
            ++qB;
          } else {
            const int s_ = static_cast<int>(pseq % nstage);
            const uint32_t use = pseq / nstage;
            if (use == 0 || mbar_try_wait(&empty[s_], (use - 1) & 1u)) {
              const int ld = q_ld[qB];
              const int KC = max(4, (slot / ld) & ~3);
              const int kc = min(KC, ld - ck0);
              const uint32_t bytes = static_cast<uint32_t>(kc) * ld * 8u;
              fence_proxy_async_smem();
              mbar_arrive_expect_tx(&full[s_], bytes);
              tma_load_1d(ring + s_ * slot, B + q_boff[qB] + static_cast<int64_t>(ck0) * ld, bytes, &full[s_]);
              ++pseq;
              ck0 += KC;
              if (ck0 >= ld) { ck0 = 0; ++qB; }
            }
          }
        }
      }
    }
    return;
  }
  // ============================ consumers ============================
  const int qr = lane >> 2, qc = lane & 3;
  uint32_t seq = 0;
  unsigned long long tsm[1 + 3 * MAXQ];
  int nts = 0;
  auto stamp = [&]() {
    if ((a.dbg & 16) && tid == 0 && nts < 1 + 3 * MAXQ) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tsm[nts++] = tt;
    }
  };
  stamp();
  for (int q = 0; q < nmine; ++q) {
    const int t = blockIdx.x + q * G;
    const int ld = q_ld[q];
    const int64_t p0 = q_p0[q];
    const int mtt = ld >> 3;
    // 1. D_i from stgD (fused: D = R + beta o P_old for active columns, P_new written back)
    mbar_wait(&dbar, static_cast<uint32_t>(q & 1));
    for (int idx = tid; idx < ld * 9; idx += NWM * 32) {
      const int c = idx / ld, k = idx - c * ld;
      double v = stgD[c * ld + k];
      if (a.fuse_p) {
        const double po = stgD[(9 + c) * ld + k];
        v = (cb[NCPE + c] != 0.0) ? v + cb[c] * po : po;
        Pnew[c * n_pad + p0 + k] = v;
      }
      if (c == 0) ys[k] = v; else Dp[k * LDP + (c - 1)] = v;
    }
    mma_sync_consumers();
    stamp();
    if (tid == 0) mbar_arrive(&dfree);
    // 2. block term: DMMA over the ring chunks
    double acc0[MTMAX], acc1[MTMAX], accy[MTMAX];
#pragma unroll
    for (int j = 0; j < MTMAX; ++j) { acc0[j] = 0.0; acc1[j] = 0.0; accy[j] = 0.0; }
    if (useB) {
      const int KC = max(4, (slot / ld) & ~3);
      for (int k0 = 0; k0 < ld; k0 += KC, ++seq) {
        const int kc = min(KC, ld - k0);
        const int s_ = static_cast<int>(seq % nstage);
        mbar_wait(&full[s_], (seq / nstage) & 1u);
        const double* cbuf = ring + s_ * slot;
        if (!(a.dbg & 1)) {
          for (int kq = 0; kq < kc; kq += 4) {
            const int k = k0 + kq + qc;
            const double bfr = Dp[k * LDP + qr];
            const double yv = ys[k];
            const double* acol = cbuf + (kq + qc) * ld + qr;
#pragma unroll
            for (int j = 0; j < MTMAX; ++j) {
              const int mt = wid + j * NWM;
              if (mt < mtt) {
                const double afr = acol[mt * 8];
                dmma884(acc0[j], acc1[j], afr, bfr);
                accy[j] = fma(afr, yv, accy[j]);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s_]);
      }
    }
#pragma unroll
    for (int j = 0; j < MTMAX; ++j) {
      accy[j] += __shfl_xor_sync(0xffffffffu, accy[j], 1);
      accy[j] += __shfl_xor_sync(0xffffffffu, accy[j], 2);
    }
    stamp();
    // 3. epilogue from shared memory
    mbar_wait(&ebar, static_cast<uint32_t>(q & 1));
    double ep[NCPE];
#pragma unroll
    for (int c = 0; c < NCPE; ++c) ep[c] = 0.0;
    {
      const double bi = q_bi[q];
      const double pa = P->a, ms = P->mscale;
      const double* su = stgE;
      const double* sP2 = stgE + ld;                    // column c at sP2[c*ld]
      const double* sY2 = eY2 ? stgE + 10 * ld : sP2;
#pragma unroll
      for (int j = 0; j < MTMAX; ++j) {
        const int mt = wid + j * NWM;
        if (mt < mtt) {
          const int r = mt * 8 + qr;
          const double uu = su[r];
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            if (e == 2 && qc != 0) continue;
            const int c = (e < 2) ? 1 + 2 * qc + e : 0;
            const double bd = (e == 0) ? acc0[j] : (e == 1) ? acc1[j] : accy[j];
            const double d = (e < 2) ? Dp[r * LDP + c - 1] : ys[r];
            double val = pa * d;
            if (useB) val += bi * bd;
            val += uu * (ms * sT[c]);
            double o = a.cA[c] * val + a.cV[c] * d;
            if (P2) o += a.cP[c] * sP2[c * ld + r];
            a.out[c * n_pad + p0 + r] = o;
            const double y2 = (a.epi == EPI_S) ? uu : sY2[c * ld + r];
#pragma unroll
            for (int cc = 0; cc < 9; ++cc)
              if (cc == c) ep[cc] += o * y2;
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NCPE; ++c) ep[c] = warp_sum(ep[c]);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < NCPE; ++c) sred[wid * NCPE + c] = ep[c];
    }
    mma_sync_consumers();
    if (tid < ncol) {
      double s = 0.0;
      for (int w = 0; w < NWM; ++w) s += sred[w * NCPE + tid];
      if (a.epi == EPI_S) a.Sout[t * MAXC + tid] = s;
      else a.dots[t * MAXC + tid] = s;
    }
    mma_sync_consumers();                                   // sred / Dp / ys / stgE reuse
    if (tid == 0) mbar_arrive(&efree);
    stamp();
  }
  if ((a.dbg & 16) && tid == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    for (int k = 0; k < nts; ++k)
      printf("T %d %u %d %llu\n", blockIdx.x, smid, k, tsm[k]);
  }
  // 4. finaliser (last CTA among the consumers; one warp per column)
  if (a.fin != FIN_NONE) {
    __shared__ int s_last;
    __threadfence();
    mma_sync_consumers();
    if (tid == 0) {
      const unsigned int tk = atomicAdd(&a.st->ticket[a.fin], 1u);
      s_last = (tk == gridDim.x - 1);
    }
    mma_sync_consumers();
    if (s_last) {
      __threadfence();
      CGState* st = a.st;
      fin_alpha_trace_body(a.fin, st, a.dots, n_tiles, ncol, a.alpha_hist, a.hist_stride, NWM);
      mma_sync_consumers();
      if (tid == 0) st->ticket[a.fin] = 0;
    }
  }
}

// ---------------------------------------------------------------------------------------
// DMMA apply over column tasks (c = 9, ld_max <= 256; the default for C1-C3).  B_i is symmetric
// (H or G), so its columns [c0, c0+16) are also rows [c0, c0+16) and are CONTIGUOUS in the
// column-major storage: a task = (cluster i, 16 output rows) streams 16 whole columns of B_i and
// produces those rows of out completely.  Tasks (~13 per C3 cluster) are split evenly over one
// persistent CTA per SM, so all SMs stream until the end (whole-cluster work units leave 15% of
// the SMs idle at C3).  Warp NWM is the producer: per task it lands the 16 B columns (one bulk
// copy each, padded row stride lds = ld (mod 16) + 4 so the A-fragment loads are bank-conflict
// free) plus the task's epilogue inputs (u, P2, Y2 rows) in one ring slot; per cluster it lands
// the 9 D columns, the low-rank row T_i and b_i in a D slot (3-deep ring).  Consumer warp w owns
// the CTA's tasks w, w+NWM, ...; there is no CTA-wide barrier: each warp waits on its slot's
// full barrier, runs the DMMAs, writes its rows and per-task partial sums, and releases the slot.
constexpr int NDB = 3;                    // D-slot ring depth
constexpr int MAXT = 96;                  // column tasks per CTA (metadata cache)

template <int MT>   // m-tiles per task (CTW / 8)
__global__ void __launch_bounds__(NTM, 1) apply_col_kernel(ApplyArgs a) {
  constexpr int NCPE = 10;
  if (a.gate && !a.st->any_active) return;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[MAX_NSTAGE], empty[MAX_NSTAGE];
  __shared__ __align__(8) uint64_t dfull[NDB], dempty[NDB];
  __shared__ int s_task[MAX_NSTAGE], s_qseq[MAX_NSTAGE];
  __shared__ int d_ntask[NDB], d_cnt[NDB], d_ld[NDB], d_q[NDB];
  __shared__ int64_t d_p0[NDB];
  __shared__ double d_bi[NDB];
  __shared__ int tk_blk[MAXT], tk_row0[MAXT], tk_nc[MAXT], tk_ld[MAXT];
  __shared__ int64_t tk_p0[MAXT], tk_boff[MAXT];
  __shared__ double tk_bi[MAXT];
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int64_t n_pad = a.L.n_pad;
  const int ncol = a.ncol;                 // == 9
  const EvalParams* P = a.prm;
  const int par = a.st->par;
  const double* B = P->B;
  const bool useB = (B != nullptr);
  const int nstage = a.nstage;
  const int lds = a.lds;
  const int T = a.L.n_ctasks;
  const int G = gridDim.x;
  const int t0 = static_cast<int>((static_cast<int64_t>(T) * blockIdx.x) / G);
  const int t1 = static_cast<int>((static_cast<int64_t>(T) * (blockIdx.x + 1)) / G);
  const int nt = t1 - t0;
  const double* D = a.d_is_pnew ? a.Pbuf[par ^ 1] : a.D;
  const double* P2 = a.use_par_p2 == 1 ? a.Pbuf[par ^ 1] : a.P2;
  const double* Y2 = a.use_par_p2 ? a.Pbuf[par ^ 1] : a.Y2;
  // slot layout (doubles): task slot = CTW columns of B_i at their natural stride ld (one bulk copy)
  const int tslot = CTW * a.ld_max;
  const int dslot = 9 * lds + 16;                              // 9 D columns | T_i (16)
  double* ring = sm;
  double* dring = ring + nstage * tslot;
  if (tid == 0) {
    for (int s_ = 0; s_ < nstage; ++s_) { mbar_init(&full[s_], 1); mbar_init(&empty[s_], 1); s_task[s_] = -1; }
    for (int s_ = 0; s_ < NDB; ++s_) { mbar_init(&dfull[s_], 1); mbar_init(&dempty[s_], 1); d_cnt[s_] = 0; d_q[s_] = -1; }
    fence_mbar_init();
  }
  // task metadata of this CTA, loaded once (the plan guarantees nt <= MAXT)
  for (int j = tid; j < nt; j += NTM) {
    const TileDesc td = a.L.ctasks[t0 + j];
    tk_blk[j] = td.blk;
    tk_row0[j] = td.row0;
    tk_nc[j] = td.nrows;
    tk_ld[j] = a.L.ld[td.blk];
    tk_p0[j] = a.L.poff[td.blk];
    tk_boff[j] = a.L.boff[td.blk];
    tk_bi[j] = P->b0 + P->b1 * a.jitter[td.blk];
  }
  __syncthreads();
  if (wid == NWM) {
    // ============================ producer warp ============================
    int qseq = -1, cur = -1;
    for (int j = 0; j < nt; ++j) {
      const int i = tk_blk[j];
      const int ld = tk_ld[j];
      const int64_t p0 = tk_p0[j];
      const uint32_t cb8 = static_cast<uint32_t>(ld) * 8u;
      if (i != cur) {                                          // new cluster: D slot
        cur = i;
        ++qseq;
        const int ds = qseq % NDB;
        if (qseq >= NDB) mbar_wait(&dempty[ds], static_cast<uint32_t>((qseq / NDB - 1) & 1));
        double* dst = dring + ds * dslot;
        if (lane == 0) {
          int cnt = 0;
          for (int jj = j; jj < nt && tk_blk[jj] == i; ++jj) ++cnt;
          d_ntask[ds] = cnt;
          d_ld[ds] = ld;
          d_p0[ds] = p0;
          d_bi[ds] = tk_bi[j];
          *reinterpret_cast<volatile int*>(&d_q[ds]) = qseq;
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&dfull[ds], cb8 * 9u + 16u * 8u);
        }
        __syncwarp();
        if (lane < 9) tma_load_1d(dst + lane * lds, D + lane * n_pad + p0, cb8, &dfull[ds]);
        else if (lane == 9) tma_load_1d(dst + 9 * lds, a.Tbuf + static_cast<int64_t>(i) * MAXC, 16u * 8u, &dfull[ds]);
      }
      const int s_ = j % nstage;
      if (j >= nstage) mbar_wait(&empty[s_], static_cast<uint32_t>((j / nstage - 1) & 1));
      const int nc = tk_nc[j];
      if (lane == 0) {
        s_qseq[s_] = qseq;
        *reinterpret_cast<volatile int*>(&s_task[s_]) = t0 + j;
        if (useB) {
          const uint32_t bytes = cb8 * static_cast<uint32_t>(nc);
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full[s_], bytes);
          tma_load_1d(ring + s_ * tslot, B + tk_boff[j] + static_cast<int64_t>(tk_row0[j]) * ld, bytes, &full[s_]);
        } else {
          mbar_arrive(&full[s_]);
        }
      }
      __syncwarp();
    }
    return;
  }
  // ============================ consumer warps ============================
  const int qr = lane >> 2, qc = lane & 3;
  const double pa = P->a, ms = P->mscale;
  for (int j = wid; j < nt; j += NWM) {
    const int s_ = j % nstage;
    // A warp's first use of a slot may be the slot's k-th: a parity wait is only meaningful once
    // the producer has started that use (it publishes the task id first), else the "previous
    // phase" of a fresh barrier would satisfy it.  Same for the D slots.
    while (*reinterpret_cast<volatile int*>(&s_task[s_]) != t0 + j) __nanosleep(64);
    mbar_wait(&full[s_], static_cast<uint32_t>((j / nstage) & 1));
    const int gt = t0 + j;
    const int qs = s_qseq[s_];
    const int ds = qs % NDB;
    while (*reinterpret_cast<volatile int*>(&d_q[ds]) != qs) __nanosleep(64);
    mbar_wait(&dfull[ds], static_cast<uint32_t>((qs / NDB) & 1));
    const double* tsl = ring + s_ * tslot;
    const double* dsl = dring + ds * dslot;
    const int ld = d_ld[ds];
    const int64_t p0 = d_p0[ds];
    TileDesc td;
    td.blk = tk_blk[j]; td.row0 = tk_row0[j]; td.nrows = tk_nc[j];
    const int nmt = td.nrows >> 3;
    // epilogue inputs (global, issued now so their latency hides behind the DMMA loop)
    double uu[MT], p2v[MT][3], y2v[MT][3];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const bool on = m < nmt;
      const int r = td.row0 + m * 8 + qr;
      uu[m] = on ? __ldg(a.u + p0 + r) : 0.0;
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        const int c = (e < 2) ? 1 + 2 * qc + e : 0;
        const int64_t gi = c * n_pad + p0 + r;
        const bool le = on && (e < 2 || qc == 0);
        p2v[m][e] = (le && P2) ? P2[gi] : 0.0;
        y2v[m][e] = (le && a.epi != EPI_S) ? Y2[gi] : 0.0;
      }
    }
    double acc0[MT], acc1[MT], accy[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) { acc0[m] = 0.0; acc1[m] = 0.0; accy[m] = 0.0; }
    if (useB && !(a.dbg & 1)) {
      const double* bcol = dsl + (1 + qr) * lds + qc;           // B fragment: D[k][n = qr]
      const double* ycol = dsl + qc;
      const double* arow = tsl + qr * ld + qc;                  // A fragment: B_i[k][r = qr] (row r = column)
#pragma unroll 4
      for (int k0 = 0; k0 < ld; k0 += 4) {
        const double bfr = bcol[k0];
        const double yv = ycol[k0];
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          if (m < nmt) {
            const double afr = arow[m * 8 * ld + k0];
            dmma884(acc0[m], acc1[m], afr, bfr);
            accy[m] = fma(afr, yv, accy[m]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s_]);                     // B columns consumed: slot free
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      accy[m] += __shfl_xor_sync(0xffffffffu, accy[m], 1);
      accy[m] += __shfl_xor_sync(0xffffffffu, accy[m], 2);
    }
    // epilogue: lane owns row m*8 + qr of the task, probe columns 1 + 2qc + {0,1}, y if qc == 0
    double ep[NCPE];
#pragma unroll
    for (int c = 0; c < NCPE; ++c) ep[c] = 0.0;
    const double bi = d_bi[ds];
    const double* sT = dsl + 9 * lds;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (m < nmt) {
        const int r = td.row0 + m * 8 + qr;                     // row within the cluster
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          if (e == 2 && qc != 0) continue;
          const int c = (e < 2) ? 1 + 2 * qc + e : 0;
          const double bd = (e == 0) ? acc0[m] : (e == 1) ? acc1[m] : accy[m];
          const double d = dsl[c * lds + r];
          double val = pa * d;
          if (useB) val += bi * bd;
          val += uu[m] * (ms * sT[c]);
          double o = a.cA[c] * val + a.cV[c] * d;
          if (P2) o += a.cP[c] * p2v[m][e];
          a.out[c * n_pad + p0 + r] = o;
          const double y2 = (a.epi == EPI_S) ? uu[m] : y2v[m][e];
#pragma unroll
          for (int cc = 0; cc < 9; ++cc)
            if (cc == c) ep[cc] += o * y2;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) ep[c] = warp_sum(ep[c]);
    double* part = (a.epi == EPI_S) ? a.Sout : a.dots;
    if (lane < 9) {
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < 9; ++c) if (c == lane) v = ep[c];
      part[static_cast<int64_t>(gt) * MAXC + lane] = v;
    }
    __syncwarp();
    if (lane == 0) {
      if (atomicAdd(&d_cnt[ds], 1) + 1 == d_ntask[ds]) {        // last task of this cluster's D slot
        d_cnt[ds] = 0;
        mbar_arrive(&dempty[ds]);
      }
    }
  }
  // finaliser (last CTA; one warp per column)
  if (a.fin != FIN_NONE) {
    __shared__ int s_last;
    __threadfence();
    mma_sync_consumers();
    if (tid == 0) {
      const unsigned int tk = atomicAdd(&a.st->ticket[a.fin], 1u);
      s_last = (tk == gridDim.x - 1);
    }
    mma_sync_consumers();
    if (s_last) {
      __threadfence();
      CGState* st = a.st;
      for (int c = wid; c < ncol; c += NWM) {
        const double tot = col_total(a.dots, T, c);
        if (lane == 0) {
          if (a.fin == FIN_ALPHA) {
            if (st->active[c]) {
              const double al = st->rr[c] / tot;          // alpha = r^T r / p^T q
              st->alpha[c] = al;
              a.alpha_hist[c * a.hist_stride + st->iters[c]] = al;
            }
          } else {  // FIN_TRACE
            if (c == 0) st->quad = tot; else st->t[c] = tot;
          }
        }
      }
      mma_sync_consumers();
      if (tid == 0) st->ticket[a.fin] = 0;
    }
  }
}

// P_new = R + beta o P_old for the active columns (P_old kept for frozen ones): the fused
// search-direction update of the first apply, run as its own pass for the column-task apply.
__global__ void __launch_bounds__(NT) pnew_kernel(const CGState* st, const double* R, double* const* Pbuf_unused,
                                                  const double* P0, const double* P1, double* Q0, double* Q1,
                                                  int64_t n_pad, int ncol) {
  (void)Pbuf_unused;
  const int par = st->par;
  const double* Pold = par ? P1 : P0;
  double* Pnew = par ? Q0 : Q1;
  const int64_t tot = n_pad * ncol;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(NT) + threadIdx.x; g < tot; g += static_cast<int64_t>(gridDim.x) * NT) {
    const int c = static_cast<int>(g / n_pad);
    const double po = Pold[g];
    Pnew[g] = st->active[c] ? R[g] + st->beta[c] * po : po;
  }
}

// ---------------------------------------------------------------------------------------
// Low-rank coefficients T = M' S(D) (Eq. 19-21: block i of W M' W^T D is u_i T_i), one warp per
// row i, S staged once per CTA in shared memory.  With fuse_p, S(D) = S(P_new) = S(R) +
// beta o S(P_old) for the active columns (S is linear), and CTA 0 also stores S(P_new).
constexpr int TROWS = 8;   // rows of T per CTA (one per warp; 16 = two per warp measured slower at C3)

template <int NCP>
__global__ void __launch_bounds__(NT, 2) lowrank_kernel(LowrankArgs a) {
  if (a.gate && !a.st->any_active) return;
  extern __shared__ double Ss[];          // n_c * NCP
  __shared__ double cb[2 * NCP];
  const int n_c = a.n_c;
  const int ncol = a.ncol;
  const int par = a.st->par;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < NCP) {
    cb[tid] = (tid < ncol) ? a.st->beta[tid] : 0.0;
    cb[NCP + tid] = (tid < ncol) ? static_cast<double>(a.st->active[tid]) : 0.0;
  }
  __syncthreads();
  const double* SPo = a.fuse_p ? a.SPbuf[par] : nullptr;
  // stage S (n_c rows of NCP) with all loads of a thread in flight: thread -> rows j = tid + k*NT
  for (int j0 = 0; j0 < n_c; j0 += NT * 2) {
    double v[2][NCP];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = j0 + u * NT + tid;
#pragma unroll
      for (int c2 = 0; c2 < NCP / 2; ++c2) {
        double2 x = make_double2(0.0, 0.0);
        if (j < n_c) {
          if (a.task0) {         // per-column-task partials of the cluster, summed in task order
            for (int tk = a.task0[j]; tk < a.task0[j + 1]; ++tk) {
              const double2 w = *reinterpret_cast<const double2*>(a.S + tk * MAXC + 2 * c2);
              x.x += w.x;
              x.y += w.y;
            }
          } else {
            x = *reinterpret_cast<const double2*>(a.S + j * MAXC + 2 * c2);
          }
          if (a.fuse_p) {
            const double2 y = *reinterpret_cast<const double2*>(SPo + j * MAXC + 2 * c2);
            x.x = (cb[NCP + 2 * c2] != 0.0) ? x.x + cb[2 * c2] * y.x : y.x;
            x.y = (cb[NCP + 2 * c2 + 1] != 0.0) ? x.y + cb[2 * c2 + 1] * y.y : y.y;
          }
        }
        v[u][2 * c2] = x.x;
        v[u][2 * c2 + 1] = x.y;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = j0 + u * NT + tid;
      if (j < n_c) {
#pragma unroll
        for (int c = 0; c < NCP; ++c) Ss[j * NCP + c] = v[u][c];
        if (a.fuse_p && blockIdx.x == 0)
#pragma unroll
          for (int c = 0; c < NCP; ++c)
            if (c < ncol) a.SPbuf[par ^ 1][j * MAXC + c] = v[u][c];
      }
    }
  }
  __syncthreads();
  // each warp forms TROWS / 8 rows of T (one S staging per CTA serves all of them)
  for (int q = 0; q < TROWS / 8; ++q) {
    const int il = blockIdx.x * TROWS + q * 8 + wid;   // row of T (local to this rank's clusters)
    if (il >= a.nrows) return;
    const int i = a.row0 + il;                         // row of M'
    const double* Mrow = (a.prm ? a.prm->Mp : a.Mp) + static_cast<int64_t>(i) * n_c;
    double t[NCP];
#pragma unroll
    for (int c = 0; c < NCP; ++c) t[c] = 0.0;
#pragma unroll 4
    for (int j = lane; j < n_c; j += 32) {
      const double m = Mrow[j];
      const double2* sj = reinterpret_cast<const double2*>(Ss + j * NCP);
#pragma unroll
      for (int c2 = 0; c2 < NCP / 2; ++c2) {
        const double2 v = sj[c2];
        t[2 * c2] = fma(m, v.x, t[2 * c2]);
        t[2 * c2 + 1] = fma(m, v.y, t[2 * c2 + 1]);
      }
    }
#pragma unroll
    for (int c = 0; c < NCP; ++c) t[c] = warp_sum(t[c]);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < NCP; ++c) a.T[il * MAXC + c] = t[c];
    }
  }
}

// ---------------------------------------------------------------------------------------
// CG update: x += alpha p, r -= alpha q (active columns); partials of r^T r and S(r);
// the last CTA forms beta = r'^T r' / r^T r, records it, advances counters and freezes.
template <int NCP>
__global__ void __launch_bounds__(NT, 2) update_kernel(UpdateArgs a) {
  CGState* st = a.st;
  if (!st->any_active) {
    // nothing left to do: end the graph's CG while-loop (no-op outside a graph)
    if (a.cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.cond, 0u);
    return;
  }
  __shared__ double sred[(NT / 32) * MAXC];
  __shared__ double outv[MAXC];
  __shared__ double cal[NCP], cact[NCP];
  const int t = blockIdx.x;
  const TileDesc td = a.L.tiles[t];
  const int i = td.blk;
  const int64_t p0 = a.L.poff[i] + td.row0, n_pad = a.L.n_pad;
  const int ncol = a.ncol;
  const int par = st->par;
  const double* Pc = a.Pbuf[par ^ 1];
  if (threadIdx.x < NCP) {
    cal[threadIdx.x] = (threadIdx.x < ncol) ? st->alpha[threadIdx.x] : 0.0;
    cact[threadIdx.x] = (threadIdx.x < ncol) ? static_cast<double>(st->active[threadIdx.x]) : 0.0;
  }
  __syncthreads();
  double rr[NCP], sr[NCP];
#pragma unroll
  for (int c = 0; c < NCP; ++c) { rr[c] = 0.0; sr[c] = 0.0; }
  for (int rl = threadIdx.x; rl < td.nrows; rl += NT) {
    const int64_t g = p0 + rl;
    const double uu = a.u[g];
    double xv[NCP], pv[NCP], rv[NCP], qv[NCP];
#pragma unroll
    for (int c = 0; c < NCP; ++c) {
      const bool on = c < ncol && cact[c] != 0.0;
      const int64_t gi = c * n_pad + g;
      xv[c] = on ? a.X[gi] : 0.0;
      pv[c] = on ? Pc[gi] : 0.0;
      rv[c] = on ? a.R[gi] : 0.0;
      qv[c] = on ? a.Q[gi] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < NCP; ++c) {
      if (c < ncol && cact[c] != 0.0) {
        const int64_t gi = c * n_pad + g;
        const double al = cal[c];
        a.X[gi] = xv[c] + al * pv[c];
        const double r2 = rv[c] - al * qv[c];
        a.R[gi] = r2;
        rr[c] += r2 * r2;
        sr[c] += uu * r2;
      }
    }
  }
  block_reduce_cols<NCP>(rr, sred, outv);
  if (threadIdx.x < ncol) a.rr_part[t * MAXC + threadIdx.x] = outv[threadIdx.x];
  __syncthreads();
  block_reduce_cols<NCP>(sr, sred, outv);
  if (threadIdx.x < ncol) a.SR_part[t * MAXC + threadIdx.x] = outv[threadIdx.x];
  if (!a.nofin && last_cta(&st->ticket[FIN_UPDATE])) {
    fin_update_body(st, a.prm, a.rr_part, a.L.n_tiles, ncol, a.beta_hist, a.hist_stride, a.cond, NT / 32);
    if (threadIdx.x == 0) st->ticket[FIN_UPDATE] = 0;
  }
}

// ---------------------------------------------------------------------------------------
// S partials of a vector block: part[t][c] = sum_rows u * V[c]  (used before the trace applies)
__global__ void __launch_bounds__(NT) spart_kernel(LayoutDev L, const double* u, const double* V,
                                                   int ncol, double* part) {
  __shared__ double sred[(NT / 32) * MAXC];
  __shared__ double outv[MAXC];
  const TileDesc td = L.tiles[blockIdx.x];
  const int64_t p0 = L.poff[td.blk] + td.row0;
  double s[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) s[c] = 0.0;
  for (int rl = threadIdx.x; rl < td.nrows; rl += NT) {
    const double uu = u[p0 + rl];
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < ncol) s[c] += uu * V[c * L.n_pad + p0 + rl];
  }
  block_reduce_cols<MAXC>(s, sred, outv);
  if (threadIdx.x < MAXC) part[blockIdx.x * MAXC + threadIdx.x] = outv[threadIdx.x];
}

// ---------------------------------------------------------------------------------------
// final: SLQ per probe (thread j), Pade log-det, MLL assembly into a nugpr_mll_out record.
struct FinalArgs {
  const CGState* st;
  const EvalParams* prm;
  const double* alpha_hist;
  const double* beta_hist;
  int hist_stride;
  double* slq_work;          // [MAXC][3*hist_stride]
  const double* logdet_R;    // device scalar
  double n;
  int ncol;
  int logdet_mode;
  nugpr_mll_out* out;
  const double* quad_part;   // NEXT-4 (mBCG): partials of c^T x (column 0), summed in order
  int n_quad_part;
};

__global__ void final_kernel(FinalArgs a) {
  __shared__ double s_slq[MAXC];
  const CGState* st = a.st;
  const int j = threadIdx.x;
  if (j >= 1 && j < a.ncol) {
    const int k = st->iters[j];
    double val = 0.0;
    if (k > 0) {
      // the usual k (<= 64 CG iterations) in shared memory; long histories in the global scratch
      __shared__ double sh_dez[MAXC][3][64];
      double* d = a.slq_work + static_cast<int64_t>(j) * 3 * a.hist_stride;
      double* e = d + a.hist_stride;
      double* z = e + a.hist_stride;
      if (k <= 64) { d = sh_dez[j][0]; e = sh_dez[j][1]; z = sh_dez[j][2]; }
      const double* al = a.alpha_hist + j * a.hist_stride;
      const double* be = a.beta_hist + j * a.hist_stride;
      d[0] = 1.0 / al[0];
      for (int q = 1; q < k; ++q) d[q] = 1.0 / al[q] + be[q - 1] / al[q - 1];
      for (int q = 0; q + 1 < k; ++q) e[q] = sqrt(be[q]) / al[q];
      tql_first(k, d, e, z);
      if (a.logdet_mode == 2)            // mBCG on A: Ritz values of A itself, f = log
        for (int l = 0; l < k; ++l) val += z[l] * z[l] * log(d[l]);
      else                               // CG on Q(A): map mu -> lambda = -2 + sqrt(3 + mu)
        for (int l = 0; l < k; ++l) val += z[l] * z[l] * log(-2.0 + sqrt(3.0 + d[l]));
      val *= st->rr0[j];
    }
    s_slq[j] = val;
  }
  __syncthreads();
  if (j == 0) {
    const int m = a.ncol - 1;
    double tsum = 0.0, ssum = 0.0, rq = 0.0;
    int kq = 0;
    nugpr_mll_out o;
    for (int q = 0; q < 16; ++q) { o.iters_q[q] = 0; o.probe_t[q] = 0.0; o.probe_s[q] = 0.0; }
    for (int c = 1; c < a.ncol; ++c) {
      tsum += st->t[c];
      ssum += s_slq[c];
      rq = fmax(rq, sqrt(st->rr[c]));
      kq = max(kq, st->iters[c]);
      o.iters_q[c - 1] = st->iters[c];
      o.probe_t[c - 1] = (a.logdet_mode == 2) ? __longlong_as_double(0x7ff8000000000000ll) : st->t[c];
      o.probe_s[c - 1] = s_slq[c];
    }
    const double ldR = a.logdet_R[0];
    if (a.quad_part) {
      double q = 0.0;
      for (int b = 0; b < a.n_quad_part; ++b) q += a.quad_part[b];
      o.quad = q;
    } else {
      o.quad = st->quad;
    }
    o.logdet_R = ldR;
    o.logdet_pade = (a.logdet_mode == 2) ? __longlong_as_double(0x7ff8000000000000ll) : ldR + tsum / m;
    o.logdet_slq = ldR + ssum / m;
    o.logdet = (a.logdet_mode != 0) ? o.logdet_slq : o.logdet_pade;
    o.L = 0.5 * (o.quad + o.logdet + a.n * 1.8378770664093453);   // n log(2 pi)
    o.lambda0 = a.prm->lam0_src ? a.prm->lam0_src[0] * a.prm->lam0_mul : a.prm->lam0_val;
    o.resid_y = sqrt(st->rr[0]);
    o.resid_q_max = rq;
    o.iters_y = st->iters[0];
    o.iters_q_max = kq;
    o.converged = (st->hit_max || st->breakdown) ? 0 : 1;
    o.mode = a.prm->mode;
    o.breakdown = st->breakdown;
    o.lanczos_iters = a.prm->lz_info ? a.prm->lz_info[0] : 0;
    o.lanczos_converged = a.prm->lz_info ? a.prm->lz_info[1] : 1;
    o.lambda0_degenerate = a.prm->lz_info ? a.prm->lz_info[2] : 0;
    *a.out = o;
  }
}

// NEXT-4 (mBCG): quad = c^T x over column 0, per-CTA partials of contiguous ranges (fixed order)
__global__ void __launch_bounds__(256) quad_part_kernel(const double* c, const double* x, int64_t n_pad,
                                                        int64_t chunk, double* part) {
  __shared__ double red[8];
  const int64_t lo = blockIdx.x * chunk, hi = min(n_pad, lo + chunk);
  double s = 0.0;
  for (int64_t p = lo + threadIdx.x; p < hi; p += 256) s = fma(c[p], x[p], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------------------
// probe export (debug): Z[j][p] for the seed, cluster-sorted order
__global__ void probe_gen_kernel(uint64_t seed, int m, int64_t n, double* Z) {
  int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(m) * n) return;
  int j = static_cast<int>(idx / n);
  int64_t p = idx % n;
  Z[idx] = probe_value(seed, j, p);
}

// ======================================================================================
// launchers
static int num_sms() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

// Shared-memory plan of the apply kernel (host side): ring depth chosen to fit.
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

int num_sms_host() { return num_sms(); }

// FP32-stored copy of a block array (NUGPR_F32_BLOCKS): round to nearest
__global__ void d2f_kernel(const double* src, float* dst, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = __double2float_rn(src[k]);
}
void launch_d2f(const double* src, float* dst, int64_t n, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 8 * num_sms()));
  d2f_kernel<<<grid, 256, 0, s>>>(src, dst, n);
  note_launch(); post_launch("d2f_kernel");
}

// Shared-memory / grid plan of the apply (host side).  ncol == 9 (the paper's m = 8) uses the DMMA
// kernel unless NUGPR_APPLY_MMA=0; the ring depth is chosen to fit; NUGPR_APPLY_{SLOT,PER,BAL}
// are tuning knobs (slot doubles, max CTAs per SM, equal clusters per CTA).
ApplyPlan plan_apply(int ncp, int ncol, int ld_max, int ld_min, int n_tiles, int grid_unused, int n_ctasks) {
  (void)grid_unused;
  int dev = 0, optin = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  const bool mma = (ncol == 9) && env_int("NUGPR_APPLY_MMA", 1) != 0;
  const size_t fixed = mma ? static_cast<size_t>(ld_max) * (LDP + 1)
                           : static_cast<size_t>(2) * ncol * ld_max + static_cast<size_t>(ld_max) * ncp +
                                 static_cast<size_t>(NWC) * ncp + 3 * ncp;
  const size_t static_smem = 4096;   // static shared memory + the 1 KB per-CTA system reservation, with margin
  const int slot_target = env_int("NUGPR_APPLY_SLOT", SLOT_TARGET_DOUBLES);
  const int per_max = std::max(1, std::min(3, env_int("NUGPR_APPLY_PER", 2)));
  const bool balance = env_int("NUGPR_APPLY_BAL", 1) != 0;
  const int col_mode = env_int("NUGPR_APPLY_COL", 0);     // experimental (slower at C3 so far)
  if (mma && col_mode && ld_max <= 256) {
    ApplyPlan p;
    p.mma = 3;
    p.lds = ld_max + ((4 - ld_max % 16) + 16) % 16;             // lds = 4 (mod 16)
    const size_t tslot = static_cast<size_t>(CTW) * ld_max;
    const size_t dslot = static_cast<size_t>(9) * p.lds + 16;
    const size_t budget = static_cast<size_t>(optin) - 8192;
    p.ctas_per_sm = 1;
    p.grid = num_sms();
    p.slot_doubles = static_cast<int>(tslot);
    const long avail = static_cast<long>(budget / sizeof(double)) - static_cast<long>(NDB * dslot);
    p.nstage = static_cast<int>(std::min<long>(MAX_NSTAGE, avail / static_cast<long>(tslot)));
    p.smem_nob = p.smem_b = (NDB * dslot + static_cast<size_t>(std::max(p.nstage, 0)) * tslot) * sizeof(double);
    p.ok = p.nstage >= 3 && (n_ctasks + p.grid - 1) / p.grid <= MAXT;
    if (p.ok) return p;
  }
  const int stage_mode = env_int("NUGPR_APPLY_STAGE", 0); // experimental (no gain at C3 so far)
  if (mma && stage_mode) {
    for (int per = std::min(per_max, 2); per >= 1; --per) {
      ApplyPlan p;
      p.mma = 2;
      const size_t fixed_s = static_cast<size_t>(ld_max) * (18 + 19 + LDP + 1) + 16;
      const size_t budget = std::min<size_t>(static_cast<size_t>(optin), static_cast<size_t>(per_sm) / per) - 8192;
      p.ctas_per_sm = per;
      p.grid = std::min(n_tiles, per * num_sms());
      p.nmine_max = (n_tiles + p.grid - 1) / p.grid;
      if (balance) p.grid = (n_tiles + p.nmine_max - 1) / p.nmine_max;
      p.slot_doubles = std::max(per == 2 ? std::min(slot_target, 2048) : slot_target, 4 * ld_max);
      const long avail = static_cast<long>(budget / sizeof(double)) - static_cast<long>(fixed_s);
      p.nstage = static_cast<int>(std::min<long>(MAX_NSTAGE, avail / p.slot_doubles));
      p.smem_nob = fixed_s * sizeof(double);
      p.smem_b = (fixed_s + static_cast<size_t>(std::max(p.nstage, 0)) * p.slot_doubles) * sizeof(double);
      p.ok = p.nstage >= (per == 2 ? 2 : 3) && p.nmine_max <= MAXQ;
      if (p.ok) return p;
    }
  }
  // experimental (NUGPR_APPLY_SMALL=1): 4 CTAs per SM of 3 consumer warps each, one cluster per
  // CTA, ld <= 216.  Measured at C3: apply 57.3 us (ncu) vs 54.7 us for the 2-CTA/SM kernel, and
  // numgrad 7.15 vs 6.65 ms — the per-cluster phases of co-resident CTAs run in lockstep, so more
  // CTAs do not overlap them (profiles/r01i_apply_small_ab.txt)
  if (mma && ld_max <= 9 * NW_SMALL * 8 && env_int("NUGPR_APPLY_SMALL", 0) != 0) {
    ApplyPlan p;
    p.mma = 1;
    p.nw = NW_SMALL;
    const int per = 4;
    const size_t budget = std::min<size_t>(static_cast<size_t>(optin), static_cast<size_t>(per_sm) / per) - static_smem;
    p.ctas_per_sm = per;
    p.grid = std::min(n_tiles, per * num_sms());
    p.nmine_max = (n_tiles + p.grid - 1) / p.grid;
    p.slot_doubles = std::max(env_int("NUGPR_APPLY_SLOT_SMALL", 4 * ld_max), 4 * ld_max);
    const long avail = static_cast<long>(budget / sizeof(double)) - static_cast<long>(fixed);
    p.nstage = static_cast<int>(std::min<long>(MAX_NSTAGE, avail / p.slot_doubles));
    p.smem_nob = fixed * sizeof(double);
    p.smem_b = (fixed + static_cast<size_t>(std::max(p.nstage, 0)) * p.slot_doubles) * sizeof(double);
    p.ok = p.nstage >= 2;
    if (p.ok) return p;
  }
  for (int per = per_max; per >= 1; --per) {
    ApplyPlan p;
    p.mma = mma ? 1 : 0;
    p.nw = NWM;
    const size_t budget = std::min<size_t>(static_cast<size_t>(optin), static_cast<size_t>(per_sm) / per) - static_smem;
    p.red_doubles = 0;
    p.ctas_per_sm = per;
    p.grid = std::min(n_tiles, per * num_sms());
    p.nmine_max = (n_tiles + p.grid - 1) / p.grid;
    if (balance) p.grid = (n_tiles + p.nmine_max - 1) / p.nmine_max;
    p.slot_doubles = std::max(slot_target, mma ? 4 * ld_max : ld_max);
    // progressive D (DMMA apply): per stage also 18 rows-of-chunk of D / P_old, row stride dstride
    // (the largest chunk width over the clusters for FP32 or FP64 blocks, + 2 against bank conflicts)
    const bool prog = mma && env_int("NUGPR_APPLY_PROG", 0) != 0;   // experimental: slower at C3 (profiles/r01i_apply_prog_sweep.txt)
    auto dstride_for = [&](int slot) { return prog ? std::max(4, (2 * slot / std::max(ld_min, 8)) & ~3) + 2 : 0; };
    p.dstride = dstride_for(p.slot_doubles);
    long avail = static_cast<long>(budget / sizeof(double)) - static_cast<long>(fixed);
    p.nstage = static_cast<int>(std::min<long>(MAX_NSTAGE, avail / (p.slot_doubles + 18 * p.dstride)));
    if (p.nstage < 2) {
      p.slot_doubles = mma ? 4 * ld_max : ld_max;
      p.dstride = dstride_for(p.slot_doubles);
      p.nstage = static_cast<int>(std::min<long>(MAX_NSTAGE, avail / (p.slot_doubles + 18 * p.dstride)));
    }
    p.smem_nob = fixed * sizeof(double);
    p.smem_b = (fixed + static_cast<size_t>(std::max(p.nstage, 0)) * (p.slot_doubles + 18 * p.dstride)) *
               sizeof(double);
    const int dbuf_mode = env_int("NUGPR_APPLY_DBUF", 1);   // 2: measured slower at C3 (smaller ring slot)
    if (mma && dbuf_mode >= 1) {
      // second D_i buffer (next-cluster prefetch) if the ring keeps the same number of stages
      const long avail2 = avail - static_cast<long>(fixed);
      const int ns2 = static_cast<int>(std::min<long>(MAX_NSTAGE, avail2 / (p.slot_doubles + 18 * p.dstride)));
      if (ns2 >= 2 && ns2 == p.nstage) {
        p.dbuf = 1;
        p.smem_nob = 2 * fixed * sizeof(double);
        p.smem_b = (2 * fixed + static_cast<size_t>(ns2) * (p.slot_doubles + 18 * p.dstride)) * sizeof(double);
      }
      // + a P_old staging area so the fused apply prefetches too, trading at most 1/4 of the ring slot
      const long fixed3 = 2 * static_cast<long>(fixed) + 9L * ld_max;
      const long avail3 = static_cast<long>(budget / sizeof(double)) - fixed3;
      const int slot3 = std::min<int>(p.slot_doubles, static_cast<int>(avail3 / 2));
      if (dbuf_mode >= 2 && p.dbuf && p.dstride == 0 && slot3 >= 4 * ld_max && 4 * slot3 >= 3 * p.slot_doubles) {
        p.dbuf = 2;
        p.slot_doubles = slot3;
        p.nstage = static_cast<int>(std::min<long>(MAX_NSTAGE, avail3 / slot3));
        p.smem_nob = fixed3 * sizeof(double);
        p.smem_b = (fixed3 + static_cast<size_t>(p.nstage) * p.slot_doubles) * sizeof(double);
      }
    }
    p.ok = p.nstage >= 2;
    if (p.ok) return p;
  }
  return ApplyPlan();
}

int apply_grid(int n_tiles) { return std::min(n_tiles, 2 * num_sms()); }

template <int NCP>
static void apply_launch_t(const ApplyArgs& a, bool useB, cudaStream_t s) {
  size_t smem = useB ? a.smem_b : a.smem_nob;
  smem_optin(reinterpret_cast<const void*>(apply_kernel<NCP>));
  apply_kernel<NCP><<<a.grid, NTA, smem, s>>>(a);
  note_launch(); post_launch("apply_kernel");
}

void launch_apply(const ApplyArgs& a, int ncp, bool useB, cudaStream_t s) {
  if (a.big) { launch_apply_big(a, ncp, s); return; }
  if (a.mma == 3) {
    size_t smem = a.smem_b;
    smem_optin(reinterpret_cast<const void*>(apply_col_kernel<CTW / 8>));
    apply_col_kernel<CTW / 8><<<a.grid, NTM, smem, s>>>(a);
    note_launch(); post_launch("apply_col_kernel");
    return;
  }
  if (a.mma == 2) {
    size_t smem = useB ? a.smem_b : a.smem_nob;
    if (a.ld_max <= 4 * NWM * 8) {
      smem_optin(reinterpret_cast<const void*>(apply_mma_staged_kernel<4>));
      apply_mma_staged_kernel<4><<<a.grid, NTM, smem, s>>>(a);
    } else if (a.ld_max <= 8 * NWM * 8) {
      smem_optin(reinterpret_cast<const void*>(apply_mma_staged_kernel<8>));
      apply_mma_staged_kernel<8><<<a.grid, NTM, smem, s>>>(a);
    } else {
      smem_optin(reinterpret_cast<const void*>(apply_mma_staged_kernel<10>));
      apply_mma_staged_kernel<10><<<a.grid, NTM, smem, s>>>(a);
    }
    note_launch(); post_launch("apply_mma_staged_kernel");
    return;
  }
  if (a.mma) {
    size_t smem = useB ? a.smem_b : a.smem_nob;
#define NUGPR_AMK(MT, TBT)                                                                  \
  do {                                                                                      \
    smem_optin(reinterpret_cast<const void*>(apply_mma_kernel<MT, TBT, NWM>));             \
    apply_mma_kernel<MT, TBT, NWM><<<a.grid, NTM, smem, s>>>(a);                           \
  } while (0)
    if (a.nw == NW_SMALL) {
      if (a.f32) {
        smem_optin(reinterpret_cast<const void*>(apply_mma_kernel<9, float, NW_SMALL>));
        apply_mma_kernel<9, float, NW_SMALL><<<a.grid, (NW_SMALL + 1) * 32, smem, s>>>(a);
      } else {
        smem_optin(reinterpret_cast<const void*>(apply_mma_kernel<9, double, NW_SMALL>));
        apply_mma_kernel<9, double, NW_SMALL><<<a.grid, (NW_SMALL + 1) * 32, smem, s>>>(a);
      }
    } else if (a.ld_max <= 4 * NWM * 8) {
      if (a.f32) NUGPR_AMK(4, float); else NUGPR_AMK(4, double);
    } else if (a.ld_max <= 8 * NWM * 8) {
      if (a.f32) NUGPR_AMK(8, float); else NUGPR_AMK(8, double);
    } else {
      if (a.f32) NUGPR_AMK(10, float); else NUGPR_AMK(10, double);
    }
#undef NUGPR_AMK
    note_launch(); post_launch("apply_mma_kernel");
    return;
  }
  switch (ncp) {
    case 2: apply_launch_t<2>(a, useB, s); break;
    case 4: apply_launch_t<4>(a, useB, s); break;
    case 6: apply_launch_t<6>(a, useB, s); break;
    case 8: apply_launch_t<8>(a, useB, s); break;
    case 10: apply_launch_t<10>(a, useB, s); break;
    case 12: apply_launch_t<12>(a, useB, s); break;
    case 14: apply_launch_t<14>(a, useB, s); break;
    default: apply_launch_t<16>(a, useB, s); break;
  }
}

template <int NCP>
static void lowrank_launch_t(const LowrankArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(double) * static_cast<size_t>(a.n_c) * NCP;
  smem_optin(reinterpret_cast<const void*>(lowrank_kernel<NCP>));
  lowrank_kernel<NCP><<<(a.nrows + TROWS - 1) / TROWS, NT, smem, s>>>(a);
  note_launch(); post_launch("lowrank_kernel");
}

void launch_lowrank(const LowrankArgs& a, int ncp, cudaStream_t s) {
  switch (ncp) {
    case 2: lowrank_launch_t<2>(a, s); break;
    case 4: lowrank_launch_t<4>(a, s); break;
    case 6: lowrank_launch_t<6>(a, s); break;
    case 8: lowrank_launch_t<8>(a, s); break;
    case 10: lowrank_launch_t<10>(a, s); break;
    case 12: lowrank_launch_t<12>(a, s); break;
    case 14: lowrank_launch_t<14>(a, s); break;
    default: lowrank_launch_t<16>(a, s); break;
  }
}

void launch_update(const UpdateArgs& a, int ncp, cudaStream_t s) {
  switch (ncp) {
    case 2: update_kernel<2><<<a.L.n_tiles, NT, 0, s>>>(a); note_launch(); post_launch("update_kernel"); break;
    case 4: update_kernel<4><<<a.L.n_tiles, NT, 0, s>>>(a); note_launch(); post_launch("update_kernel"); break;
    case 6: update_kernel<6><<<a.L.n_tiles, NT, 0, s>>>(a); note_launch(); post_launch("update_kernel"); break;
    case 8: update_kernel<8><<<a.L.n_tiles, NT, 0, s>>>(a); note_launch(); post_launch("update_kernel"); break;
    case 10: update_kernel<10><<<a.L.n_tiles, NT, 0, s>>>(a); note_launch(); post_launch("update_kernel"); break;
    case 12: update_kernel<12><<<a.L.n_tiles, NT, 0, s>>>(a); note_launch(); post_launch("update_kernel"); break;
    case 14: update_kernel<14><<<a.L.n_tiles, NT, 0, s>>>(a); note_launch(); post_launch("update_kernel"); break;
    default: update_kernel<16><<<a.L.n_tiles, NT, 0, s>>>(a); note_launch(); post_launch("update_kernel"); break;
  }
}

void launch_rhs_init(const RhsArgs& a, int ld_max, cudaStream_t s) {
  size_t smem = sizeof(double) * (static_cast<size_t>(ld_max) + NT * MAXC + MAXC);
  smem_optin(reinterpret_cast<const void*>(rhs_init_kernel));
  rhs_init_kernel<<<a.L.n_tiles, NT, smem, s>>>(a);
  note_launch(); post_launch("rhs_init_kernel");
}

void launch_cy(const LayoutDev& L, const double* Linv, const double* y, int ld_max, double* cy, cudaStream_t s) {
  cy_kernel<<<L.n_tiles, NT, sizeof(double) * ld_max, s>>>(L, Linv, y, cy);
  note_launch(); post_launch("cy_kernel");
}

void launch_apply_multi(const ApplyArgs* ga, int ng, cudaStream_t s) {
  MultiApplyArgs ma;
  memset(&ma, 0, sizeof(ma));
  for (int g = 0; g < ng; ++g) ma.g[g] = ga[g];
  ma.ng = ng;
  const ApplyArgs& a = ga[0];
  const size_t smem = a.smem_b;
#define NUGPR_AM(MT, NGV)                                                                   \
  do {                                                                                      \
    smem_optin(reinterpret_cast<const void*>(apply_multi_kernel<MT, NGV>));                \
    apply_multi_kernel<MT, NGV><<<a.grid, NTM, smem, s>>>(ma);                             \
  } while (0)
  if (a.ld_max <= 4 * NWM * 8) {
    if (ng == 2) NUGPR_AM(4, 2); else if (ng == 3) NUGPR_AM(4, 3); else if (ng == 4) NUGPR_AM(4, 4); else NUGPR_AM(4, 1);
  } else {
    if (ng == 2) NUGPR_AM(10, 2); else if (ng == 3) NUGPR_AM(10, 3); else if (ng == 4) NUGPR_AM(10, 4); else NUGPR_AM(10, 1);
  }
#undef NUGPR_AM
  note_launch(); post_launch("apply_multi_kernel");
}

size_t apply_multi_smem(int ng, int ld_max, int slot_doubles, int nstage) {
  const int ldg = (ng == 1) ? 12 : (ng == 2) ? 20 : 36;
  return sizeof(double) * (static_cast<size_t>(nstage) * slot_doubles + static_cast<size_t>(ld_max) * (ldg + ng));
}

void launch_cond_any(const CGState* const* sts, int ng, unsigned long long cond, cudaStream_t s) {
  cond_any_kernel<<<1, 1, 0, s>>>(sts[0], ng > 1 ? sts[1] : sts[0], ng > 2 ? sts[2] : sts[0], ng > 3 ? sts[3] : sts[0],
                                  ng, cond);
  note_launch(); post_launch("cond_any_kernel");
}

void launch_pnew(const CGState* st, const double* R, double* const* Pbuf, int64_t n_pad, int ncol, cudaStream_t s) {
  const int64_t tot = n_pad * ncol;
  const int grid = static_cast<int>(std::min<int64_t>((tot + NT - 1) / NT, 4 * num_sms()));
  pnew_kernel<<<grid, NT, 0, s>>>(st, R, nullptr, Pbuf[0], Pbuf[1], Pbuf[0], Pbuf[1], n_pad, ncol);
  note_launch(); post_launch("pnew_kernel");
}

void launch_spart(const LayoutDev& L, const double* u, const double* V, int ncol, double* part,
                  cudaStream_t s) {
  spart_kernel<<<L.n_tiles, NT, 0, s>>>(L, u, V, ncol, part);
  note_launch(); post_launch("spart_kernel");
}

int quad_parts(int64_t n_pad, int cap) {
  const int64_t want = (n_pad + 4095) / 4096;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({want, static_cast<int64_t>(num_sms()), cap})));
}

void launch_quad_part(const double* c, const double* x, int64_t n_pad, int nparts, double* part, cudaStream_t s) {
  const int64_t chunk = (n_pad + nparts - 1) / nparts;
  quad_part_kernel<<<nparts, 256, 0, s>>>(c, x, n_pad, chunk, part);
  note_launch(); post_launch("quad_part_kernel");
}

void launch_final(const CGState* st, const EvalParams* prm, const double* ah, const double* bh,
                  int stride, double* slq_work, const double* logdet_R, double n,
                  int ncol, int logdet_mode, nugpr_mll_out* out, cudaStream_t s,
                  const double* quad_part, int n_quad_part) {
  FinalArgs a{st, prm, ah, bh, stride, slq_work, logdet_R, n, ncol, logdet_mode, out, quad_part, n_quad_part};
  final_kernel<<<1, 32, 0, s>>>(a);
  note_launch(); post_launch("final_kernel");
}

void launch_fin(int fin, CGState* st, const EvalParams* prm, const double* part, int n_tiles, int ncol,
                double* hist, int hist_stride, cudaStream_t s) {
  fin_kernel<<<1, NT, 0, s>>>(fin, st, prm, part, n_tiles, ncol, hist, hist_stride);
  note_launch(); post_launch("fin_kernel");
}

void launch_probe_gen(uint64_t seed, int m, int64_t n, double* Z, cudaStream_t s) {
  int64_t tot = static_cast<int64_t>(m) * n;
  probe_gen_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(seed, m, n, Z);
  note_launch(); post_launch("probe_gen_kernel");
}

}  // namespace nugpr
