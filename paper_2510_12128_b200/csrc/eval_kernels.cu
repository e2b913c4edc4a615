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

#include "cg_fin.cuh"
#include "common.cuh"
#include "kernels_decl.h"
#include "tma.cuh"
#include "tridiag.h"

namespace nugpr {

// PAR-2 (cluster-sharded evaluation): the finaliser as its own single-CTA launch
// after the exchange of the partials.  FIN_UPDATE skips when no column is active (as update does).
__global__ void __launch_bounds__(NT) fin_kernel(int fin, CGState* st, const EvalParams* prm, const double* part,
                                                 int n_tiles, int ncol, double* hist, int hist_stride, SPUpdate sp,
                                                 unsigned long long cond) {
  if (fin == FIN_INIT) {
    fin_init_body(st, prm, part, n_tiles, ncol, NT / 32);
  } else if (fin == FIN_UPDATE) {
    if (!st->any_active) {                       // (graph mode: end the CG while-loop)
      if (cond && threadIdx.x == 0) cudaGraphSetConditional(cond, 0u);
      return;
    }
    fin_update_body(st, prm, part, n_tiles, ncol, hist, hist_stride, cond, NT / 32, sp);
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
  const bool per_cluster = a.L.n_tiles == a.L.n_c;   // (big layout: several tiles per cluster)
  if (threadIdx.x < MAXC) {
    a.SR_part[t * MAXC + threadIdx.x] = outv[threadIdx.x];
    if (per_cluster) a.SP0[t * MAXC + threadIdx.x] = outv[threadIdx.x];   // S(P_0) = S(R_0)
  }
  if (!a.nofin && last_cta(&a.st->ticket[FIN_INIT])) {
    fin_init_body(a.st, a.prm, a.rr_part, a.L.n_tiles, ncol, NT / 32);
    if (!per_cluster)                                // S(P_0) rows: the cluster's tiles in tile order
      for (int idx = threadIdx.x; idx < a.L.n_c * MAXC; idx += NT) {
        const int j = idx / MAXC, c = idx - j * MAXC;
        double x = 0.0;
        for (int tt = a.L.tile0[j]; tt < a.L.tile0[j + 1]; ++tt) x += a.SR_part[tt * MAXC + c];
        a.SP0[idx] = x;
      }
    if (threadIdx.x == 0) a.st->ticket[FIN_INIT] = 0;
  }
}

// ---------------------------------------------------------------------------------------
// Low-rank coefficients T = M' S(D) (Eq. 19-21: block i of W M' W^T D is u_i T_i) for the
// big-block layout's apply (the packed apply forms its rows in-kernel), one warp per
// row i, S staged once per CTA in shared memory.  With fuse_p, S(D) = S(P_new), the rows the update
// finaliser (or rhs_init) formed in SPbuf[par].
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
          if (a.fuse_p) {        // S(P_new) rows, formed by the update finaliser
            x = *reinterpret_cast<const double2*>(a.SPbuf[par] + j * MAXC + 2 * c2);
          } else if (a.task0) {  // per-column-task partials of the cluster, summed in task order
            for (int tk = a.task0[j]; tk < a.task0[j + 1]; ++tk) {
              const double2 w = *reinterpret_cast<const double2*>(a.S + tk * MAXC + 2 * c2);
              x.x += w.x;
              x.y += w.y;
            }
          } else {
            x = *reinterpret_cast<const double2*>(a.S + j * MAXC + 2 * c2);
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
  __shared__ double sred2[(NT / 32) * 2 * NCP];
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
  // both per-tile partial rows (r^T r and S(r)) in one pass: warp butterflies, one barrier, then the
  // warps in fixed order (the same sums as two block_reduce_cols passes)
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < NCP; ++c) { rr[c] = warp_sum(rr[c]); sr[c] = warp_sum(sr[c]); }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < NCP; ++c) { sred2[wid * 2 * NCP + c] = rr[c]; sred2[wid * 2 * NCP + NCP + c] = sr[c]; }
    }
    __syncthreads();
    if (threadIdx.x < 2 * NCP) {
      const int v = threadIdx.x, c = v % NCP;
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += sred2[w * 2 * NCP + v];
      if (c < ncol) (v < NCP ? a.rr_part : a.SR_part)[t * MAXC + c] = s;
    }
  }
  if (!a.nofin && last_cta(&st->ticket[FIN_UPDATE])) {
    SPUpdate sp{a.SR_part, a.L.n_tiles == a.L.n_c ? nullptr : a.L.tile0, a.L.n_c, {a.SPbuf[0], a.SPbuf[1]}};
    fin_update_body(st, a.prm, a.rr_part, a.L.n_tiles, ncol, a.beta_hist, a.hist_stride, a.cond, NT / 32, sp);
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

int num_sms_host() { return num_sms(); }

// FP32-stored copy of a block array (NUGPR_BLOCKS_F32, reading X6): round to nearest
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

// The apply: packed-block DMMA kernel for the small layout (apply_kernels.cu), the row-tiled
// kernel on full blocks for the big-block layout (big_kernels.cu).
void launch_apply(const ApplyArgs& a, int ncp, cudaStream_t s) {
  if (a.big) launch_apply_big(a, ncp, s);
  else launch_apply_packed(a, s);
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
                double* hist, int hist_stride, cudaStream_t s, const double* SR, double* SP0, double* SP1,
                unsigned long long cond) {
  SPUpdate sp{SR, nullptr, n_tiles, {SP0, SP1}};
  fin_kernel<<<1, NT, 0, s>>>(fin, st, prm, part, n_tiles, ncol, hist, hist_stride, sp, cond);
  note_launch(); post_launch("fin_kernel");
}

void launch_probe_gen(uint64_t seed, int m, int64_t n, double* Z, cudaStream_t s) {
  int64_t tot = static_cast<int64_t>(m) * n;
  probe_gen_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(seed, m, n, Z);
  note_launch(); post_launch("probe_gen_kernel");
}

}  // namespace nugpr
