// cg_fin.cuh — block reductions and the CG finalisers shared by the evaluation kernels.
//
// Every global reduction of the method (S = W^T D, p^T q, r^T r, the Pade trace dots) is written as
// per-cluster (per-tile) partial rows [n][MAXC] and summed in fixed order by ONE CTA — the last CTA
// of the kernel that wrote them, or fin_kernel after a PAR-2 exchange — so results are
// bit-reproducible (no floating-point atomics).  The finalisers implement the CG scalar recurrences
// of PAPER.md:107-108 / 124 with readings P3-P5 (absolute tol per column, x0 = 0, per-column
// alpha/beta, freezing) and the breakdown guard (non-finite or non-positive curvature).
#pragma once
#include "common.cuh"

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
static __device__ void fin_init_body(CGState* st, const EvalParams* prm, const double* rr_part, int n_tiles, int ncol,
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
// nw warps take part: warps w0 .. w0+nw-1 of the CTA.
__device__ __forceinline__ void fin_alpha_trace_body(int fin, CGState* st, const double* dots, int n_tiles,
                                                     int ncol, double* alpha_hist, int hist_stride, int nw,
                                                     int w0 = 0) {
  const int lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) - w0;
  if (wid < 0 || wid >= nw) return;
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

// S(P) rows of the next search direction, formed where beta is decided (so the next fused apply
// reads them ready-made): S(P_{k+1}) = S(R_{k+1}) + beta o S(P_k) on active columns, S(P_k) on frozen
// ones (S = W^T . is linear, Eq. 19-21).  SR: per-tile S(r) rows; tile0 (or NULL: one tile per cluster)
// maps cluster j to its tiles, summed in tile order.
struct SPUpdate {
  const double* SR;
  const int32_t* tile0;
  int n_c;
  double* SP[2];
};

// FIN_UPDATE: beta = r'^T r' / r^T r, history, iteration counters, freezing (readings P3, P5).
static __device__ void fin_update_body(CGState* st, const EvalParams* P, const double* rr_part, int n_tiles, int ncol,
                                double* beta_hist, int hist_stride, unsigned long long cond, int nw,
                                const SPUpdate& sp) {
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
  if (sp.SR) {
    // all CTA threads, 16-byte rows pairs, eight loads of each in flight before the stores
    __shared__ double sbeta[MAXC];
    __shared__ int sact[MAXC];
    if (threadIdx.x < MAXC) {
      const int c = threadIdx.x;
      sact[c] = (c < ncol) ? act[c] : 0;
      sbeta[c] = (c < ncol && act[c]) ? st->beta[c] : 0.0;
    }
    __syncthreads();
    const double2* SPo2 = reinterpret_cast<const double2*>(sp.SP[par]);
    double2* SPn2 = reinterpret_cast<double2*>(sp.SP[par ^ 1]);
    const double2* SR2 = reinterpret_cast<const double2*>(sp.SR);
    const int tot = sp.n_c * (MAXC / 2);
    constexpr int U = 8;
    for (int base = threadIdx.x; base < tot; base += U * blockDim.x) {
      double2 y[U], x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * blockDim.x;
        y[u] = make_double2(0.0, 0.0);
        x[u] = make_double2(0.0, 0.0);
        if (idx < tot) {
          y[u] = SPo2[idx];
          if (sp.tile0) {
            const int j = idx / (MAXC / 2), h = idx - j * (MAXC / 2);
            for (int t = sp.tile0[j]; t < sp.tile0[j + 1]; ++t) {
              const double2 w = SR2[static_cast<int64_t>(t) * (MAXC / 2) + h];
              x[u].x += w.x;
              x[u].y += w.y;
            }
          } else {
            x[u] = SR2[idx];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * blockDim.x;
        if (idx < tot) {
          const int c0 = 2 * (idx % (MAXC / 2));
          double2 v;
          v.x = sact[c0] ? x[u].x + sbeta[c0] * y[u].x : y[u].x;
          v.y = sact[c0 + 1] ? x[u].y + sbeta[c0 + 1] * y[u].y : y[u].y;
          SPn2[idx] = v;
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    int any = 0;
    for (int c = 0; c < ncol; ++c) any |= act[c];
    st->any_active = any;
    st->par = par ^ 1;
    if (cond) cudaGraphSetConditional(cond, any ? 1u : 0u);
  }
}

}  // namespace nugpr
