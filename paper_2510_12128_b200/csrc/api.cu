// api.cu — C-ABI entry points and host orchestration of the nuGPR hot path.
//
// Host code here only marshals arguments, carves the caller's workspace, enqueues kernels on
// the context stream and runs the tiny host-side steps the paper keeps on the host (the
// halving decisions of Alg. 1 and the Adam update).  Every step of the MLL
// evaluation runs in the CUDA kernels of build_kernels.cu / eval_kernels.cu.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/nugpr.h"
#include "common.cuh"
#include "nccl_rt.h"
#include "kernels_decl.h"
#include "tridiag.h"

using namespace nugpr;

namespace {

thread_local std::string g_err;

nugpr_status fail(nugpr_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) return fail(NUGPR_ERR_CUDA, "%s: %s (%s:%d)", #call,       \
                                       cudaGetErrorString(e_), __FILE__, __LINE__);   \
  } while (0)

#define CKL()                                                                         \
  do {                                                                                \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess) return fail(NUGPR_ERR_CUDA, "kernel launch: %s (%s:%d)",   \
                                       cudaGetErrorString(e_), __FILE__, __LINE__);   \
  } while (0)

#define RET(expr)                                  \
  do {                                             \
    nugpr_status s_ = (expr);                      \
    if (s_ != NUGPR_OK) return s_;                 \
  } while (0)

constexpr int HIST = 4096;          // max recorded CG iterations (cg_max_iter cap)
constexpr int LD_MAX_SUPPORTED = 8192;
constexpr int LD_SMALL_MAX = 512;     // above: big-block mode (blocked multi-launch factorisation, row-tiled apply)
// Lanczos iteration cap for lambda_0: with full reorthogonalisation, k = n_c iterations reproduce the
// whole spectrum, so the cap only binds (and the solve reports non-convergence) for n_c > 2048.
constexpr int LANCZOS_KMAX_CAP = 2048;

struct HostLayout {
  int n_c = 0, d = 0;
  bool big = false;
  int64_t n = 0, n_pad = 0, blk_total = 0;
  int64_t pk_total = 0;           // packed symmetric storage of H / G (small layout): 64 sum tri(mt_i)
  int ld_max = 0;
  std::vector<int64_t> off, poff, boff, pboff;
  std::vector<int32_t> ld, tile0;
  std::vector<TileDesc> tiles;
  // packed-apply partition (small layout): pieces of the packed stream per CTA, split scratch
  std::vector<SegDesc> segs;
  std::vector<int32_t> seg0;
  int seg_max = 0, n_split = 0;
  int64_t split_doubles = 0;
};

// Cut the packed tile stream of all clusters (blocks in storage order, cluster after cluster) into at
// most PACK_CTAS pieces of (nearly) equal tile count: whole clusters where a cluster fits one CTA's
// share, else at block boundaries; a block (whole cluster) goes to the CTA whose range holds its
// midpoint.  Clusters may span several CTAs (<= MAX_PARTS; the target
// grows until that holds).  The partition depends only on the offsets (not on the device).
static void make_partition(HostLayout& L) {
  const int n_c = L.n_c;
  int64_t total = 0;
  for (int i = 0; i < n_c; ++i) total += tri_tiles(L.ld[i] / 8);
  int G = static_cast<int>(std::min<int64_t>(PACK_CTAS, std::max<int64_t>(1, total / 64)));
  for (;; G = std::max(1, G * 3 / 4)) {
    L.segs.clear();
    L.seg0.clear();
    std::vector<int> parts(n_c, 0);
    int64_t cum = 0;
    int cur = -1;
    for (int i = 0; i < n_c; ++i) {
      const int mt = L.ld[i] / 8, ns = pk_ns(mt);
      int bi = 0;
      int64_t loc = 0;                               // tiles of cluster i before block bi (storage order)
      for (int sb = 0; sb < ns; ++sb)
        for (int gb = sb; gb < ns; ++gb, ++bi) {
          const int64_t len = pk_blk_size(gb, sb, mt);
          // a cluster of up to two CTA shares stays whole (its CTA is the one holding its midpoint; CTAs
          // left without work are not launched): a split costs a global combine and a second epilogue
          // chain (C3: 818 vs 748 evals/s whole; C2, 1.5 shares per cluster: 2391 vs 1823); larger
          // clusters are cut at block boundaries
          const int64_t ctot = tri_tiles(mt);
          const bool whole = ctot * G <= 2 * total;        // <= 2 shares (C2: 2391 vs 1823 evals/s at 1)
          const int cta = whole ? (bi == 0 ? static_cast<int>(std::min<int64_t>(G - 1, (2 * cum + ctot) * G / (2 * total))) : cur)
                                : static_cast<int>(std::min<int64_t>(G - 1, (2 * cum + len) * G / (2 * total)));
          const SegDesc fresh{i, bi, bi + 1, 0, 0, -1, 0, L.pboff[i] / 64 + loc, static_cast<int32_t>(len), 0};
          if (cta != cur) {                          // a new CTA starts here
            L.seg0.push_back(static_cast<int32_t>(L.segs.size()));
            cur = cta;
            L.segs.push_back(fresh);
            L.segs.back().part = parts[i]++;
          } else if (L.segs.back().blk != i) {       // same CTA, next cluster
            L.segs.push_back(fresh);
            L.segs.back().part = parts[i]++;
          } else {
            L.segs.back().k1 = bi + 1;
            L.segs.back().ntile += static_cast<int32_t>(len);
          }
          cum += len;
          loc += len;
        }
    }
    L.seg0.push_back(static_cast<int32_t>(L.segs.size()));
    int pmax = 0;
    for (int i = 0; i < n_c; ++i) pmax = std::max(pmax, parts[i]);
    if (pmax <= MAX_PARTS || G == 1) {
      // split scratch: nparts_i x ld_i x 17 doubles per split cluster (17 = y + 16 probe slots)
      L.n_split = 0;
      L.split_doubles = 0;
      std::vector<int> tick(n_c, -1);
      std::vector<int64_t> sp(n_c, 0);
      for (int i = 0; i < n_c; ++i) {
        if (parts[i] > 1) {
          tick[i] = L.n_split++;
          sp[i] = L.split_doubles;
          L.split_doubles += static_cast<int64_t>(parts[i]) * L.ld[i] * 17;
        }
      }
      for (SegDesc& sd : L.segs) {
        sd.nparts = parts[sd.blk];
        sd.tick = tick[sd.blk];
        sd.spoff = sp[sd.blk];
      }
      L.seg_max = 0;
      for (size_t b = 0; b + 1 < L.seg0.size(); ++b) L.seg_max = std::max(L.seg_max, L.seg0[b + 1] - L.seg0[b]);
      return;
    }
  }
}

nugpr_status make_layout(const int64_t* offsets, int n_c, int d, HostLayout& L) {
  if (!offsets) return fail(NUGPR_ERR_INVALID_ARG, "offsets is NULL");
  if (n_c < 1) return fail(NUGPR_ERR_INVALID_ARG, "n_c must be >= 1");
  if (d < 1 || d > 32) return fail(NUGPR_ERR_INVALID_ARG, "d must be in [1, 32]");
  if (offsets[0] != 0) return fail(NUGPR_ERR_SHAPE, "offsets[0] must be 0");
  L = HostLayout();
  L.n_c = n_c;
  L.d = d;
  L.off.assign(offsets, offsets + n_c + 1);
  int64_t bmax = 0;
  for (int i = 0; i < n_c; ++i) bmax = std::max<int64_t>(bmax, offsets[i + 1] - offsets[i]);
  L.big = (bmax + PAD - 1) / PAD * PAD > LD_SMALL_MAX;
  const int tile_rows = L.big ? 64 : TILE_ROWS;
  L.poff.resize(n_c + 1);
  L.boff.resize(n_c);
  L.pboff.resize(n_c);
  L.ld.resize(n_c);
  L.tile0.resize(n_c + 1);
  int64_t pp = 0, bb = 0, pk = 0;
  for (int i = 0; i < n_c; ++i) {
    int64_t b = offsets[i + 1] - offsets[i];
    if (b <= 0) return fail(NUGPR_ERR_SHAPE, "offsets must be strictly increasing (cluster %d empty)", i);
    int64_t ld = (b + PAD - 1) / PAD * PAD;
    if (ld > LD_MAX_SUPPORTED)
      return fail(NUGPR_ERR_SHAPE, "cluster %d has %lld points; this build supports <= %d per cluster",
                  i, (long long)b, LD_MAX_SUPPORTED);
    L.ld[i] = static_cast<int32_t>(ld);
    L.ld_max = std::max<int>(L.ld_max, static_cast<int>(ld));
    L.poff[i] = pp;
    L.boff[i] = bb;
    L.pboff[i] = pk;
    L.tile0[i] = static_cast<int32_t>(L.tiles.size());
    for (int r0 = 0; r0 < ld; r0 += tile_rows) {
      TileDesc t;
      t.blk = i;
      t.row0 = r0;
      t.nrows = static_cast<int32_t>(std::min<int64_t>(tile_rows, ld - r0));
      t.pad_ = 0;
      L.tiles.push_back(t);
    }
    pp += ld;
    bb += ld * ld;
    pk += 64 * tri_tiles(static_cast<int>(ld / 8));
  }
  L.poff[n_c] = pp;
  L.tile0[n_c] = static_cast<int32_t>(L.tiles.size());
  L.n = offsets[n_c];
  L.n_pad = pp;
  L.blk_total = bb;
  L.pk_total = pk;
  if (!L.big) make_partition(L);
  return NUGPR_OK;
}

struct Carver {
  char* base;
  size_t pos = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count) {
    pos = (pos + 255) / 256 * 256;
    T* p = base ? reinterpret_cast<T*>(base + pos) : nullptr;
    pos += count * sizeof(T);
    return p;
  }
};

// One evaluation's scratch (a "slot").
struct EvalDev {
  double* G = nullptr;        // blk_total (generic mode: K(theta') then G)
  double* T = nullptr;        // blk_total (generic mode: K Linv^T)
  double* Krep = nullptr;     // n_c^2
  double* M = nullptr;        // n_c^2
  double* v0 = nullptr;       // n_c
  double* lz = nullptr;       // lanczos scratch
  int32_t* linfo = nullptr;
  double* scal = nullptr;     // [0] lam0
  double* RHS = nullptr, *R = nullptr, *X = nullptr, *V = nullptr, *Q = nullptr, *U = nullptr;
  double* Pb[2] = {nullptr, nullptr};
  double* SR = nullptr, *SPb[2] = {nullptr, nullptr}, *SV = nullptr, *SX = nullptr, *dots = nullptr,
         *rrp = nullptr;
  EvalParams* prm = nullptr;
  CGState* st = nullptr;
  nugpr_mll_out* out = nullptr;
  double* ah = nullptr, *bh = nullptr, *slqw = nullptr;
  double* Tbuf = nullptr;     // n_c x MAXC
  double* xs = nullptr, *xr = nullptr;   // PAR-2 exchange send / recv: [3][n_c_global][MAXC] each
  double* split = nullptr;               // packed apply: partial products of split clusters
  unsigned int* split_tick = nullptr;    // and their tickets (self-resetting)
};

struct BlocksDev {
  int64_t* off = nullptr, *poff = nullptr, *boff = nullptr;
  int32_t* ld = nullptr, *tile0 = nullptr, *list = nullptr, *status = nullptr, *seg0 = nullptr;
  int64_t* pboff = nullptr;
  TileDesc* tiles = nullptr;
  SegDesc* segs = nullptr;
  double* X = nullptr, *reps = nullptr;
  double* Linv = nullptr;     // R_i^{-T}, full ld_i x ld_i (boff)
  double* H = nullptr;        // H_i = Linv_i Linv_i^T: packed (pboff) in the small layout, full (boff) when big
  float* H32 = nullptr;       // FP32-stored H (NUGPR_BLOCKS_F32), same layout as H
  double* u = nullptr, *jitter = nullptr, *logdet_blk = nullptr;
  double* scal = nullptr;     // [0] logdet_R, [1] lam0
  double* Krep = nullptr, *M = nullptr, *v0 = nullptr, *lz = nullptr;
  int32_t* linfo = nullptr;
  double* Zexport = nullptr;  // m x n (debug probe export)
  double* cy = nullptr;       // n_pad: c = R^{-T} y cached across the evaluations of one numgrad
  double* ystage = nullptr;   // n: host y staged to the device
  double* bigscr = nullptr;   // big-block mode: diagonal-block inverses + inverse-step scratch
  double* cap = nullptr;      // NEXT-1/2: capacitance C = I + M~ (ldc x ldc, ldc = n_c rounded up to 8)
  double* capscr = nullptr;   // its blocked (big-block) factorisation scratch when ldc > 512
  int64_t* pmeta = nullptr;   // predict: one-block layout of C = I + M~ (off, poff, boff, ld, loff, goff)
};

// n_cg / n_glob: the global cluster / row counts (differ from L's only for PAR-2 sharded blocks,
// where L is this rank's cluster range): the representatives, K_rep, M, lambda_0 scratch and the
// staged y are global (replicated), everything per cluster / per row is local.
void carve_all(Carver& c, const HostLayout& L, int slots, BlocksDev& B, std::vector<EvalDev>& E, int n_cg = -1,
               int64_t n_glob = -1) {
  const int n_c = L.n_c;
  if (n_cg < 0) n_cg = n_c;
  if (n_glob < 0) n_glob = L.n;
  const int64_t nt = static_cast<int64_t>(L.tiles.size());
  const int kmax = std::min(n_cg, LANCZOS_KMAX_CAP);
  const size_t lzs = lanczos_scratch_doubles(n_cg, kmax);
  B.off = c.take<int64_t>(n_c + 1);
  B.poff = c.take<int64_t>(n_c + 1);
  B.boff = c.take<int64_t>(n_c);
  B.ld = c.take<int32_t>(n_c);
  B.tile0 = c.take<int32_t>(n_c + 1);
  B.list = c.take<int32_t>(n_c);
  B.status = c.take<int32_t>(n_c);
  B.tiles = c.take<TileDesc>(nt);
  B.pboff = c.take<int64_t>(n_c);
  B.segs = c.take<SegDesc>(std::max<size_t>(1, L.segs.size()));
  B.seg0 = c.take<int32_t>(std::max<size_t>(1, L.seg0.size()));
  B.X = c.take<double>(static_cast<size_t>(L.n) * L.d);
  B.reps = c.take<double>(static_cast<size_t>(n_cg) * L.d);
  B.Linv = c.take<double>(L.blk_total);
  const int64_t hsize = L.big ? L.blk_total : L.pk_total;     // stored H / G elements
  B.H = c.take<double>(hsize);
  B.H32 = reinterpret_cast<float*>(c.take<double>((hsize + 1) / 2));
  B.u = c.take<double>(L.n_pad);
  B.jitter = c.take<double>(n_c);
  B.logdet_blk = c.take<double>(n_c);
  B.scal = c.take<double>(8);
  B.Krep = c.take<double>(static_cast<size_t>(n_cg) * n_cg);
  B.M = c.take<double>(static_cast<size_t>(n_cg) * n_cg);
  B.v0 = c.take<double>(n_cg);
  B.lz = c.take<double>(lzs);
  B.linfo = c.take<int32_t>(4);
  B.Zexport = c.take<double>(static_cast<size_t>(NUGPR_MAX_PROBES) * L.n);
  B.cy = c.take<double>(L.n_pad);
  B.ystage = c.take<double>(n_glob);
  B.pmeta = c.take<int64_t>(16);
  {
    const int ldc = (n_cg + PAD - 1) / PAD * PAD;
    B.cap = c.take<double>(static_cast<size_t>(ldc) * ldc);
    if (ldc > LD_SMALL_MAX) B.capscr = c.take<double>(big_scratch_doubles(1, ldc));
  }
  if (L.big) B.bigscr = c.take<double>(big_scratch_doubles(n_c, L.ld_max));
  E.assign(slots, EvalDev());
  const size_t vec = static_cast<size_t>(MAXC) * L.n_pad;
  for (int s = 0; s < slots; ++s) {
    EvalDev& e = E[s];
    e.G = c.take<double>(L.blk_total);
    e.T = c.take<double>(L.blk_total);
    e.Krep = c.take<double>(static_cast<size_t>(n_cg) * n_cg);
    e.M = c.take<double>(static_cast<size_t>(n_cg) * n_cg);
    e.v0 = c.take<double>(n_cg);
    e.lz = c.take<double>(lzs);
    e.linfo = c.take<int32_t>(4);
    e.scal = c.take<double>(8);
    e.RHS = c.take<double>(vec);
    e.R = c.take<double>(vec);
    e.X = c.take<double>(vec);
    e.V = c.take<double>(vec);
    e.Q = c.take<double>(vec);
    e.U = c.take<double>(vec);
    e.Pb[0] = c.take<double>(vec);
    e.Pb[1] = c.take<double>(vec);
    e.SR = c.take<double>(nt * MAXC);
    e.SPb[0] = c.take<double>(std::max<int64_t>(nt, n_cg) * MAXC);   // S(P): global under PAR-2
    e.SPb[1] = c.take<double>(std::max<int64_t>(nt, n_cg) * MAXC);
    e.SV = c.take<double>(nt * MAXC);
    e.SX = c.take<double>(nt * MAXC);
    e.dots = c.take<double>(nt * MAXC);
    e.rrp = c.take<double>(nt * MAXC);
    e.prm = c.take<EvalParams>(1);
    e.st = c.take<CGState>(1);
    e.out = c.take<nugpr_mll_out>(1);
    e.ah = c.take<double>(static_cast<size_t>(MAXC) * HIST);
    e.bh = c.take<double>(static_cast<size_t>(MAXC) * HIST);
    e.slqw = c.take<double>(static_cast<size_t>(MAXC) * 3 * HIST);
    e.Tbuf = c.take<double>(static_cast<size_t>(n_c) * MAXC);
    e.xs = c.take<double>(static_cast<size_t>(3) * n_cg * MAXC);
    e.xr = c.take<double>(static_cast<size_t>(3) * n_cg * MAXC);
    e.split = c.take<double>(std::max<int64_t>(1, L.split_doubles));
    e.split_tick = c.take<unsigned int>(std::max(1, L.n_split));
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  cudaGetLastError();
  if (e != cudaSuccess) return false;
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

// Event-based per-kernel-class profiler (bench.py's live roofline): CUDA events recorded on the
// launching stream around each launch of a class, harvested at the next host sync.
enum ProfClass { PC_APPLY_B = 0, PC_APPLY_LR = 1, PC_UPDATE = 2, PC_RHS = 3, PC_GEMM = 4, PC_CHOL = 5,
                 PC_LANCZOS = 6, PC_OTHER = 7, PC_N = 8 };
struct ProfPending { int cls; double bytes; cudaEvent_t a, b; };

struct nugpr_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  nugpr_allgather_fn ag = nullptr;
  void* ag_user = nullptr;
  nugpr_allreduce_fn ar = nullptr;       // PAR-2 cluster sharding (nugpr_ctx_set_cluster_shard)
  void* ar_user = nullptr;
  bool shard_on = false;                 // PAR-2 enabled (callback or in-library NCCL)
  ncclComm_t nccl = nullptr;             // in-library communicator (nugpr_ctx_set_nccl)
  bool shard_graph_ok = true;            // the sharded CG loop captures into a graph (NCCL)
  void* nccl_scratch = nullptr;          // 64 KB device scratch for the host-record allgather
  int32_t* h_flag = nullptr;             // pinned
  nugpr_mll_out* h_out = nullptr;        // pinned
  bool prof = false;
  std::vector<cudaEvent_t> pool;
  std::vector<ProfPending> pend;
  double acc_ms[PC_N] = {0}, acc_bytes[PC_N] = {0};
  long long acc_n[PC_N] = {0};
  // concurrent evaluations: one stream per eval slot, fork/join events, pinned staging
  cudaStream_t capture_stream = nullptr;
  cudaStream_t slot_stream[NUGPR_NUM_EVALS] = {nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[NUGPR_NUM_EVALS] = {nullptr};
  // side streams for independent work inside one slot / the build (lambda_0 Lanczos next to the
  // block factorisation or the G precompute): index NUGPR_NUM_EVALS is the build's
  cudaStream_t aux_stream[NUGPR_NUM_EVALS + 1] = {nullptr};
  cudaEvent_t ev_aux[NUGPR_NUM_EVALS + 1][2] = {{nullptr}};
  EvalParams* h_prm = nullptr;           // pinned [MAX_STAGE]
  bool use_graphs = true;                // NUGPR_OPT_GRAPHS
  // nugpr_train's deferred build: H_i = Linv_i Linv_i^T on its own stream, overlapping the
  // evaluations that do not read H (baseline, lengthscale steps); ev_h1 marks it done
  cudaStream_t h_stream = nullptr;
  cudaEvent_t ev_h0 = nullptr, ev_h1 = nullptr;
  // instantiated CG graphs keyed by (workspace, layout, slot, ncol, logdet mode)
  std::unordered_map<std::string, cudaGraphExec_t> graphs;
  std::vector<cudaGraph_t> graph_defs;
};
constexpr int MAX_STAGE = 64;

static nugpr_status ensure_aux(nugpr_ctx* c, int k) {
  if (!c->aux_stream[k]) CK(cudaStreamCreateWithFlags(&c->aux_stream[k], cudaStreamNonBlocking));
  for (int e = 0; e < 2; ++e)
    if (!c->ev_aux[k][e]) CK(cudaEventCreateWithFlags(&c->ev_aux[k][e], cudaEventDisableTiming));
  return NUGPR_OK;
}

static nugpr_status ensure_slot_streams(nugpr_ctx* c, int slots) {
  for (int k = 0; k < slots && k < NUGPR_NUM_EVALS; ++k) {
    if (!c->slot_stream[k]) CK(cudaStreamCreateWithFlags(&c->slot_stream[k], cudaStreamNonBlocking));
    if (!c->ev_join[k]) CK(cudaEventCreateWithFlags(&c->ev_join[k], cudaEventDisableTiming));
  }
  if (!c->ev_fork) CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  return NUGPR_OK;
}

static int prof_begin(nugpr_ctx* c, cudaStream_t s) {
  if (!c || !c->prof) return -1;
  ProfPending p;
  for (cudaEvent_t* ev : {&p.a, &p.b}) {
    if (!c->pool.empty()) { *ev = c->pool.back(); c->pool.pop_back(); }
    else cudaEventCreate(ev);
  }
  p.cls = PC_OTHER;
  p.bytes = 0.0;
  cudaEventRecord(p.a, s);
  c->pend.push_back(p);
  return static_cast<int>(c->pend.size()) - 1;
}
static void prof_end(nugpr_ctx* c, int idx, int cls, double bytes, cudaStream_t s) {
  if (idx < 0) return;
  ProfPending& p = c->pend[idx];
  p.cls = cls;
  p.bytes = bytes;
  cudaEventRecord(p.b, s);
}
static void prof_harvest(nugpr_ctx* c) {
  if (!c) return;
  for (ProfPending& p : c->pend) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      c->acc_ms[p.cls] += ms;
      c->acc_bytes[p.cls] += p.bytes;
      c->acc_n[p.cls] += 1;
    }
    c->pool.push_back(p.a);
    c->pool.push_back(p.b);
  }
  c->pend.clear();
}
#define PROF(ctx_, cls_, bytes_, stream_, launch_)        \
  do {                                                    \
    int pi_ = prof_begin((ctx_), (stream_));              \
    launch_;                                              \
    prof_end((ctx_), pi_, (cls_), (bytes_), (stream_));   \
  } while (0)

struct nugpr_blocks {
  nugpr_ctx* ctx = nullptr;
  HostLayout L;
  LayoutDev Ld;
  BlocksDev B;
  std::vector<EvalDev> E;
  int kind = 0;
  nugpr_theta theta0{};
  double logdet_R = 0.0, lam0 = 0.0, max_jitter = 0.0;
  std::vector<double> h_jitter;
  std::vector<int32_t> h_list;
  int last_m = 0;
  uint64_t last_seed = 0;
  const double* last_probes = nullptr;
  bool cy_ready = false;      // B.cy holds c = R^{-T} y for the current numgrad call
  const void* ws_base = nullptr;
  bool f32 = false;           // current evaluation streams FP32-stored blocks
  bool h32_ready = false;     // H32 holds the FP32 copy of H
  bool h_pending = false;     // H is being formed on ctx->h_stream (wait on ctx->ev_h1 before reading it)
  // PAR-2: this rank's cluster range of the global problem (L is the local layout)
  bool shard = false;
  int c_lo = 0, c_hi = 0, n_cg = 0;
  int64_t n_glob = 0, pos0 = 0;
};

extern "C" {

const char* nugpr_version(void) { return "nugpr-b200 0.1 (sm_100a, FP64)"; }
const char* nugpr_last_error(void) { return g_err.c_str(); }

nugpr_status nugpr_ctx_create(int device, void* cuda_stream, int rank, int world, nugpr_ctx** out) {
  if (!out) return fail(NUGPR_ERR_INVALID_ARG, "out is NULL");
  if (world < 1 || rank < 0 || rank >= world) return fail(NUGPR_ERR_INVALID_ARG, "bad rank/world");
  if (device < 0) {                       // host-only context: rank/world/allgather for host helpers
    nugpr_ctx* c = new nugpr_ctx();
    c->device = -1;
    c->rank = rank;
    c->world = world;
    *out = c;
    return NUGPR_OK;
  }
  CK(cudaSetDevice(device));
  nugpr_ctx* c = new nugpr_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  c->rank = rank;
  c->world = world;
  cudaError_t e1 = cudaMallocHost(&c->h_flag, 64);
  cudaError_t e2 = cudaMallocHost(&c->h_out, sizeof(nugpr_mll_out) * MAX_STAGE);
  cudaError_t e3 = cudaMallocHost(&c->h_prm, sizeof(EvalParams) * MAX_STAGE);
  cudaError_t e4 = cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess) {
    delete c;
    return fail(NUGPR_ERR_CUDA, "pinned host allocation failed");
  }
  *out = c;
  return NUGPR_OK;
}

nugpr_status nugpr_ctx_set_allgather(nugpr_ctx* ctx, nugpr_allgather_fn fn, void* user) {
  if (!ctx) return fail(NUGPR_ERR_INVALID_ARG, "ctx is NULL");
  ctx->ag = fn;
  ctx->ag_user = user;
  return NUGPR_OK;
}

nugpr_status nugpr_ctx_set_cluster_shard(nugpr_ctx* ctx, nugpr_allreduce_fn fn, void* user) {
  if (!ctx) return fail(NUGPR_ERR_INVALID_ARG, "ctx is NULL");
  ctx->ar = fn;
  ctx->ar_user = user;
  ctx->shard_on = fn != nullptr;
  return NUGPR_OK;
}

int32_t nugpr_ctx_sharded_graphs(const nugpr_ctx* ctx) {
  return (ctx && ctx->nccl && ctx->shard_graph_ok && ctx->use_graphs) ? 1 : 0;
}

nugpr_status nugpr_nccl_unique_id(uint8_t* id) {
  if (!id) return fail(NUGPR_ERR_INVALID_ARG, "id is NULL");
  const NcclRT& rt = nccl_rt();
  if (!rt.ok) return fail(NUGPR_ERR_UNSUPPORTED, "libnccl.so.2 not found in the process or on the loader path");
  ncclUniqueId u;
  const ncclResult_t r = rt.GetUniqueId(&u);
  if (r != ncclSuccess) return fail(NUGPR_ERR_COMM, "ncclGetUniqueId: %s", rt.GetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == NUGPR_NCCL_ID_BYTES, "NCCL unique id size");
  memcpy(id, &u, sizeof(u));
  return NUGPR_OK;
}

nugpr_status nugpr_ctx_set_nccl(nugpr_ctx* ctx, const uint8_t* id) {
  if (!ctx || !id) return fail(NUGPR_ERR_INVALID_ARG, "ctx / id is NULL");
  if (ctx->device < 0) return fail(NUGPR_ERR_INVALID_ARG, "host-only context");
  const NcclRT& rt = nccl_rt();
  if (!rt.ok) return fail(NUGPR_ERR_UNSUPPORTED, "libnccl.so.2 not found in the process or on the loader path");
  CK(cudaSetDevice(ctx->device));
  if (ctx->nccl) { rt.CommDestroy(ctx->nccl); ctx->nccl = nullptr; }
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  const ncclResult_t r = rt.CommInitRank(&ctx->nccl, ctx->world, u, ctx->rank);
  if (r != ncclSuccess) { ctx->nccl = nullptr; return fail(NUGPR_ERR_COMM, "ncclCommInitRank: %s", rt.GetErrorString(r)); }
  if (!ctx->nccl_scratch) CK(cudaMalloc(&ctx->nccl_scratch, 65536));
  return NUGPR_OK;
}

nugpr_status nugpr_ctx_set_option(nugpr_ctx* ctx, int32_t option, int32_t value) {
  if (!ctx) return fail(NUGPR_ERR_INVALID_ARG, "ctx is NULL");
  switch (option) {
    case NUGPR_OPT_GRAPHS: ctx->use_graphs = value != 0; return NUGPR_OK;
    case NUGPR_OPT_SHARD_CLUSTERS:
      if (value && !ctx->nccl && !ctx->ar)
        return fail(NUGPR_ERR_INVALID_ARG, "cluster sharding needs nugpr_ctx_set_nccl or an allreduce callback");
      ctx->shard_on = value != 0;
      return NUGPR_OK;
    default: return fail(NUGPR_ERR_INVALID_ARG, "unknown option %d", option);
  }
}

nugpr_status nugpr_ctx_set_profiling(nugpr_ctx* ctx, int32_t enable) {
  if (!ctx) return fail(NUGPR_ERR_INVALID_ARG, "ctx is NULL");
  ctx->prof = enable != 0;
  for (int k = 0; k < PC_N; ++k) { ctx->acc_ms[k] = 0; ctx->acc_bytes[k] = 0; ctx->acc_n[k] = 0; }
  return NUGPR_OK;
}

nugpr_status nugpr_ctx_profile(nugpr_ctx* ctx, int32_t cls, double* ms, double* bytes, int64_t* launches) {
  if (!ctx || cls < 0 || cls >= PC_N) return fail(NUGPR_ERR_INVALID_ARG, "bad profile query");
  cudaStreamSynchronize(ctx->stream);
  prof_harvest(ctx);
  if (ms) *ms = ctx->acc_ms[cls];
  if (bytes) *bytes = ctx->acc_bytes[cls];
  if (launches) *launches = ctx->acc_n[cls];
  return NUGPR_OK;
}

int64_t nugpr_launch_count(void) { return launch_count(); }

nugpr_status nugpr_ctx_destroy(nugpr_ctx* ctx) {
  if (!ctx) return NUGPR_OK;
  if (ctx->device < 0) { delete ctx; return NUGPR_OK; }
  for (cudaEvent_t e : ctx->pool) cudaEventDestroy(e);
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
  for (cudaGraph_t g : ctx->graph_defs) cudaGraphDestroy(g);
  for (int k = 0; k < NUGPR_NUM_EVALS; ++k) {
    if (ctx->slot_stream[k]) cudaStreamDestroy(ctx->slot_stream[k]);
    if (ctx->ev_join[k]) cudaEventDestroy(ctx->ev_join[k]);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  for (int k = 0; k <= NUGPR_NUM_EVALS; ++k) {
    if (ctx->aux_stream[k]) cudaStreamDestroy(ctx->aux_stream[k]);
    for (int e = 0; e < 2; ++e) if (ctx->ev_aux[k][e]) cudaEventDestroy(ctx->ev_aux[k][e]);
  }
  if (ctx->capture_stream) cudaStreamDestroy(ctx->capture_stream);
  if (ctx->h_stream) cudaStreamDestroy(ctx->h_stream);
  if (ctx->ev_h0) cudaEventDestroy(ctx->ev_h0);
  if (ctx->ev_h1) cudaEventDestroy(ctx->ev_h1);
  if (ctx->h_flag) cudaFreeHost(ctx->h_flag);
  if (ctx->h_out) cudaFreeHost(ctx->h_out);
  if (ctx->h_prm) cudaFreeHost(ctx->h_prm);
  if (ctx->nccl) nccl_rt().CommDestroy(ctx->nccl);
  if (ctx->nccl_scratch) cudaFree(ctx->nccl_scratch);
  delete ctx;
  return NUGPR_OK;
}

}  // extern "C"

static nugpr_status ws_size_slots(const int64_t* offsets, int32_t n_c, int32_t d, int slots, size_t* bytes) {
  HostLayout L;
  RET(make_layout(offsets, n_c, d, L));
  if (L.off[n_c] <= 0) return fail(NUGPR_ERR_SHAPE, "n must be > 0");
  Carver c(nullptr);
  BlocksDev B;
  std::vector<EvalDev> E;
  carve_all(c, L, slots, B, E);
  *bytes = c.pos + 256;
  return NUGPR_OK;
}

// PAR-2 partition: contiguous cluster ranges balanced by the streamed block bytes
// sum ld_i^2, every rank at least one cluster.
static nugpr_status shard_range_impl(const int64_t* off, int n_c, int rank, int world, int* lo, int* hi) {
  if (!off || n_c < 1 || world < 1 || rank < 0 || rank >= world) return fail(NUGPR_ERR_INVALID_ARG, "bad shard range args");
  if (n_c < world) return fail(NUGPR_ERR_SHAPE, "n_c = %d < world = %d: every rank needs a cluster", n_c, world);
  std::vector<double> cum(n_c + 1, 0.0);
  for (int i = 0; i < n_c; ++i) {
    const int64_t b = off[i + 1] - off[i];
    if (b <= 0) return fail(NUGPR_ERR_SHAPE, "offsets must be strictly increasing (cluster %d empty)", i);
    const double ld = static_cast<double>((b + PAD - 1) / PAD * PAD);
    cum[i + 1] = cum[i] + ld * ld;
  }
  std::vector<int> bd(world + 1, 0);
  bd[world] = n_c;
  for (int r = 1; r < world; ++r) {
    const double target = cum[n_c] * r / world;
    int k = static_cast<int>(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
    if (k > 0 && target - cum[k - 1] < cum[k] - target) k -= 1;
    bd[r] = std::max(bd[r - 1] + 1, std::min(k, n_c - (world - r)));
  }
  *lo = bd[rank];
  *hi = bd[rank + 1];
  return NUGPR_OK;
}

extern "C" nugpr_status nugpr_shard_range(const int64_t* offsets, int32_t n_c, int32_t rank, int32_t world,
                                          int32_t range[2]) {
  if (!range) return fail(NUGPR_ERR_INVALID_ARG, "range is NULL");
  int lo = 0, hi = 0;
  RET(shard_range_impl(offsets, n_c, rank, world, &lo, &hi));
  range[0] = lo;
  range[1] = hi;
  return NUGPR_OK;
}

static std::vector<int64_t> local_offsets(const int64_t* off, int lo, int hi) {
  std::vector<int64_t> o(hi - lo + 1);
  for (int i = lo; i <= hi; ++i) o[i - lo] = off[i] - off[lo];
  return o;
}

extern "C" nugpr_status nugpr_workspace_size_shard(const int64_t* offsets, int32_t n_c, int32_t d, int32_t eval_slots,
                                                   int32_t rank, int32_t world, size_t* bytes) {
  if (!bytes) return fail(NUGPR_ERR_INVALID_ARG, "bytes is NULL");
  if (eval_slots < 1 || eval_slots > NUGPR_NUM_EVALS) return fail(NUGPR_ERR_INVALID_ARG, "eval_slots must be in [1, 7]");
  int lo = 0, hi = 0;
  RET(shard_range_impl(offsets, n_c, rank, world, &lo, &hi));
  const std::vector<int64_t> lo_off = local_offsets(offsets, lo, hi);
  HostLayout L;
  RET(make_layout(lo_off.data(), hi - lo, d, L));
  Carver c(nullptr);
  BlocksDev B;
  std::vector<EvalDev> E;
  carve_all(c, L, eval_slots, B, E, n_c, offsets[n_c]);
  *bytes = c.pos + 256;
  return NUGPR_OK;
}

extern "C" nugpr_status nugpr_workspace_size(const int64_t* offsets, int32_t n_c, int32_t d,
                                             int32_t eval_slots, size_t* bytes) {
  if (!bytes) return fail(NUGPR_ERR_INVALID_ARG, "bytes is NULL");
  if (eval_slots < 1 || eval_slots > NUGPR_NUM_EVALS) return fail(NUGPR_ERR_INVALID_ARG, "eval_slots must be in [1, 7]");
  return ws_size_slots(offsets, n_c, d, eval_slots, bytes);
}

static bool theta_ok(const nugpr_theta& t) {
  return t.lengthscale > 0 && t.noise > 0 && t.outputscale > 0 && std::isfinite(t.lengthscale) &&
         std::isfinite(t.noise) && std::isfinite(t.outputscale);
}

// Lanczos lambda_0 of K (device n_c x n_c), warm start vinit (or NULL), writes lam0/v0/M.
static nugpr_status enqueue_lambda0(nugpr_blocks* bl, const double* K, const double* vinit, double* lz,
                                    double* lam0, double* v0, double* M, int32_t* info, cudaStream_t s) {
  const int n_c = bl->n_cg;   // K_rep is global (replicated under PAR-2)
  const int kmax = std::min(n_c, LANCZOS_KMAX_CAP);
  const cudaError_t e = launch_lanczos(K, n_c, vinit, lz, kmax, 1e-11, lam0, v0, M, info, s);
  if (e != cudaSuccess) return fail(NUGPR_ERR_CUDA, "lambda_0 Lanczos launch: %s", cudaGetErrorString(e));
  CKL();
  return NUGPR_OK;
}

// ------------------------------------------------------------------------------------------
// PAR-2 exchange helpers.  Every exchange is a sum-allreduce of a zero-padded
// global array in which each rank filled only its own clusters' slots: exact, and every rank ends
// with the partials a single GPU would hold, in the same order.
static nugpr_status xchg(nugpr_ctx* ctx, const double* send, double* recv, size_t count, cudaStream_t s) {
  if (ctx->nccl) {                        // in-library NCCL on the stream (capturable into the graph)
    const NcclRT& rt = nccl_rt();
    const ncclResult_t r = rt.AllReduce(send, recv, count, ncclFloat64, ncclSum, ctx->nccl, s);
    if (r != ncclSuccess) return fail(NUGPR_ERR_COMM, "ncclAllReduce: %s", rt.GetErrorString(r));
    return NUGPR_OK;
  }
  if (!ctx->ar) return fail(NUGPR_ERR_COMM, "sharded blocks but no allreduce callback on the context");
  if (ctx->ar(send, recv, count, static_cast<void*>(s), ctx->ar_user) != 0)
    return fail(NUGPR_ERR_COMM, "allreduce callback failed (PAR-2 exchange)");
  return NUGPR_OK;
}

// per-cluster local [n_loc][w] device array -> global [n_cg][w] (glob must not be slot 0's xs)
static nugpr_status gather_clusters(nugpr_blocks* bl, const double* loc, int w, double* glob, cudaStream_t s) {
  EvalDev& e = bl->E[0];
  const size_t tot = static_cast<size_t>(bl->n_cg) * w;
  CK(cudaMemsetAsync(e.xs, 0, sizeof(double) * tot, s));
  CK(cudaMemcpyAsync(e.xs + static_cast<size_t>(bl->c_lo) * w, loc, sizeof(double) * bl->L.n_c * w,
                     cudaMemcpyDeviceToDevice, s));
  return xchg(bl->ctx, e.xs, glob, tot, s);
}

// k host doubles from every rank -> out[world][k] on every rank (synchronises s)
static nugpr_status allgather_host(nugpr_blocks* bl, const double* mine, int k, std::vector<double>& out,
                                   cudaStream_t s) {
  nugpr_ctx* ctx = bl->ctx;
  EvalDev& e = bl->E[0];
  const size_t tot = static_cast<size_t>(ctx->world) * k;
  if (tot > static_cast<size_t>(3) * bl->n_cg * MAXC) return fail(NUGPR_ERR_INTERNAL, "exchange buffer too small");
  CK(cudaMemsetAsync(e.xs, 0, sizeof(double) * tot, s));
  CK(cudaMemcpyAsync(e.xs + static_cast<size_t>(ctx->rank) * k, mine, sizeof(double) * k, cudaMemcpyHostToDevice, s));
  RET(xchg(ctx, e.xs, e.xr, tot, s));
  out.assign(tot, 0.0);
  CK(cudaMemcpyAsync(out.data(), e.xr, sizeof(double) * tot, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return NUGPR_OK;
}

// reuse: the workspace still holds this layout, X, reps and zeroed slot partials from a previous
// build on the same arguments (nugpr_train's later epochs: it owns the workspace between them), so
// the uploads and memsets are skipped.
static nugpr_status build_impl(nugpr_ctx* ctx, const double* X_sorted, const int64_t* offsets, int32_t n_c,
                               int32_t d, const double* reps, int32_t kernel, nugpr_theta theta0, void* workspace,
                               size_t ws_bytes, nugpr_blocks** out, int32_t* failed_block, double* max_jitter,
                               bool reuse, bool defer = false);

extern "C" nugpr_status nugpr_build_blocks(nugpr_ctx* ctx, const double* X_sorted, const int64_t* offsets,
                                           int32_t n_c, int32_t d, const double* reps, int32_t kernel,
                                           nugpr_theta theta0, void* workspace, size_t ws_bytes,
                                           nugpr_blocks** out, int32_t* failed_block, double* max_jitter) {
  return build_impl(ctx, X_sorted, offsets, n_c, d, reps, kernel, theta0, workspace, ws_bytes, out, failed_block,
                    max_jitter, false);
}

static nugpr_status build_impl(nugpr_ctx* ctx, const double* X_sorted, const int64_t* offsets, int32_t n_c,
                               int32_t d, const double* reps, int32_t kernel, nugpr_theta theta0, void* workspace,
                               size_t ws_bytes, nugpr_blocks** out, int32_t* failed_block, double* max_jitter,
                               bool reuse, bool defer) {
  if (failed_block) *failed_block = -1;
  if (max_jitter) *max_jitter = 0.0;
  if (!ctx || !X_sorted || !reps || !workspace || !out) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  if (kernel < 0 || kernel > 2) return fail(NUGPR_ERR_INVALID_ARG, "bad kernel id %d", kernel);
  if (!theta_ok(theta0)) return fail(NUGPR_ERR_INVALID_ARG, "theta0 must be positive and finite");
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return fail(NUGPR_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  CK(cudaSetDevice(ctx->device));
  cudaGetLastError();   // drop stale errors left by unrelated runtime calls
  if (!offsets) return fail(NUGPR_ERR_INVALID_ARG, "offsets is NULL");
  // PAR-2: this rank keeps the contiguous cluster range [c_lo, c_hi) (local layout, local blocks)
  const bool shard = ctx->shard_on;
  int c_lo = 0, c_hi = n_c;
  std::vector<int64_t> loff;
  const int64_t* offs = offsets;
  if (shard) {
    RET(shard_range_impl(offsets, n_c, ctx->rank, ctx->world, &c_lo, &c_hi));
    loff = local_offsets(offsets, c_lo, c_hi);
    offs = loff.data();
  }
  const int nl = c_hi - c_lo;               // clusters held here (= n_c unless sharded)
  nugpr_blocks* bl = new nugpr_blocks();
  nugpr_status st = make_layout(offs, nl, d, bl->L);
  if (st != NUGPR_OK) { delete bl; return st; }
  bl->shard = shard;
  bl->c_lo = c_lo; bl->c_hi = c_hi; bl->n_cg = n_c;
  bl->n_glob = offsets[n_c]; bl->pos0 = offsets[c_lo];
  if (shard && bl->L.big) {
    delete bl;
    return fail(NUGPR_ERR_UNSUPPORTED, "cluster sharding needs clusters <= %d points", LD_SMALL_MAX);
  }
  // number of eval slots that fit
  auto need_bytes = [&](int sl) {
    Carver cz(nullptr);
    BlocksDev Bz;
    std::vector<EvalDev> Ez;
    carve_all(cz, bl->L, sl, Bz, Ez, n_c, offsets[n_c]);
    return cz.pos + 256;
  };
  int slots = 0;
  for (int s = NUGPR_NUM_EVALS; s >= 1; --s) {
    if (need_bytes(s) <= ws_bytes) { slots = s; break; }
  }
  if (slots == 0) {
    const size_t need = need_bytes(1);
    delete bl;
    return fail(NUGPR_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  }
  Carver c(workspace);
  carve_all(c, bl->L, slots, bl->B, bl->E, n_c, offsets[n_c]);
  bl->ctx = ctx;
  bl->ws_base = workspace;
  bl->kind = kernel;
  bl->theta0 = theta0;
  HostLayout& L = bl->L;
  BlocksDev& B = bl->B;
  cudaStream_t s = ctx->stream;
  LayoutDev& Ld = bl->Ld;
  Ld.off = B.off; Ld.poff = B.poff; Ld.boff = B.boff; Ld.ld = B.ld; Ld.tiles = B.tiles;
  Ld.tile0 = B.tile0; Ld.n_c = nl; Ld.n_tiles = static_cast<int32_t>(L.tiles.size());
  Ld.pboff = B.pboff; Ld.segs = B.segs; Ld.seg0 = B.seg0;
  Ld.n_seg_ctas = L.seg0.empty() ? 0 : static_cast<int32_t>(L.seg0.size() - 1); Ld.seg_max = L.seg_max;
  Ld.n = L.n; Ld.n_pad = L.n_pad;
#define CKB(call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) { delete bl; \
    return fail(NUGPR_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); } } while (0)
  if (!reuse) {
    CKB(cudaMemcpyAsync(B.off, L.off.data(), sizeof(int64_t) * (nl + 1), cudaMemcpyHostToDevice, s));
    CKB(cudaMemcpyAsync(B.poff, L.poff.data(), sizeof(int64_t) * (nl + 1), cudaMemcpyHostToDevice, s));
    CKB(cudaMemcpyAsync(B.boff, L.boff.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice, s));
    CKB(cudaMemcpyAsync(B.ld, L.ld.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, s));
    CKB(cudaMemcpyAsync(B.tile0, L.tile0.data(), sizeof(int32_t) * (nl + 1), cudaMemcpyHostToDevice, s));
    CKB(cudaMemcpyAsync(B.tiles, L.tiles.data(), sizeof(TileDesc) * L.tiles.size(), cudaMemcpyHostToDevice, s));
    CKB(cudaMemcpyAsync(B.pboff, L.pboff.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice, s));
    if (!L.segs.empty()) {
      CKB(cudaMemcpyAsync(B.segs, L.segs.data(), sizeof(SegDesc) * L.segs.size(), cudaMemcpyHostToDevice, s));
      CKB(cudaMemcpyAsync(B.seg0, L.seg0.data(), sizeof(int32_t) * L.seg0.size(), cudaMemcpyHostToDevice, s));
    }
    CKB(cudaMemcpyAsync(B.X, X_sorted + static_cast<size_t>(bl->pos0) * d, sizeof(double) * L.n * d, cudaMemcpyDefault, s));
    CKB(cudaMemcpyAsync(B.reps, reps, sizeof(double) * n_c * d, cudaMemcpyDefault, s));
    for (EvalDev& ev : bl->E) {
      const size_t np = static_cast<size_t>(L.tiles.size()) * MAXC * sizeof(double);
      for (double* p : {ev.SR, ev.SPb[0], ev.SPb[1], ev.SV, ev.SX, ev.dots, ev.rrp}) CKB(cudaMemsetAsync(p, 0, np, s));
      CKB(cudaMemsetAsync(ev.st, 0, sizeof(CGState), s));
      CKB(cudaMemsetAsync(ev.split_tick, 0, sizeof(unsigned int) * std::max(1, L.n_split), s));
    }
  }
  CKB(cudaMemsetAsync(B.jitter, 0, sizeof(double) * nl, s));
  CKB(cudaMemsetAsync(B.u, 0, sizeof(double) * L.n_pad, s));
  // K_rep(theta0), lambda_0, v_0, M depend on the representatives only: side stream, overlapped
  // with the block factorisation below
  {
    nugpr_status as_ = ensure_aux(ctx, NUGPR_NUM_EVALS);
    if (as_ != NUGPR_OK) { delete bl; return as_; }
  }
  cudaStream_t bas = ctx->prof ? s : ctx->aux_stream[NUGPR_NUM_EVALS];
  if (bas != s) {
    CKB(cudaEventRecord(ctx->ev_aux[NUGPR_NUM_EVALS][0], s));
    CKB(cudaStreamWaitEvent(bas, ctx->ev_aux[NUGPR_NUM_EVALS][0], 0));
  }
  launch_krep(B.reps, n_c, d, kernel, theta0.lengthscale, theta0.outputscale, B.Krep, bas);
  {
    nugpr_status ls;
    PROF(ctx, PC_LANCZOS, 0.0, bas, ls = enqueue_lambda0(bl, B.Krep, nullptr, B.lz, B.scal + 1, B.v0, B.M, B.linfo, bas));
    if (ls != NUGPR_OK) { delete bl; return ls; }
  }
  if (bas != s) CKB(cudaEventRecord(ctx->ev_aux[NUGPR_NUM_EVALS][1], bas));
  // A1: K_i(theta0) assembled on the fly, Cholesky + inverse, jitter ladder
  if (L.big) {
    PROF(ctx, PC_OTHER, 0.0, s,
         launch_assemble(B.X, d, Ld, nullptr, 0, L.ld_max, B.jitter, B.Linv, kernel, theta0.lengthscale,
                         theta0.noise, theta0.outputscale, s));
    PROF(ctx, PC_CHOL, 0.0, s,
         launch_big_chol_trtri(B.Linv, Ld, nullptr, 0, L.ld_max, B.status, B.logdet_blk, B.u, B.bigscr, s));
  } else {
    PROF(ctx, PC_OTHER, 0.0, s,
         launch_assemble(B.X, d, Ld, nullptr, 0, L.ld_max, B.jitter, B.Linv, kernel, theta0.lengthscale,
                         theta0.noise, theta0.outputscale, s));
    PROF(ctx, PC_CHOL, 0.0, s, launch_chol_trtri(B.Linv, Ld, nullptr, 0, L.ld_max, B.status, B.logdet_blk, B.u, s));
  }
  CKB(cudaGetLastError());
  std::vector<int32_t> hstat(nl);
  CKB(cudaMemcpyAsync(hstat.data(), B.status, sizeof(int32_t) * nl, cudaMemcpyDeviceToHost, s));
  CKB(cudaStreamSynchronize(s));
  bl->h_jitter.assign(nl, 0.0);
  const double base = 1e-8 * (theta0.outputscale + theta0.noise);   // 1e-8 * mean(diag K_i)
  int fb = -1;                                                       // global index of a failed block
  for (int t = 0; t <= 5; ++t) {
    bl->h_list.clear();
    for (int i = 0; i < nl; ++i) if (hstat[i]) bl->h_list.push_back(i);
    if (bl->h_list.empty()) break;
    if (t == 5) { fb = c_lo + bl->h_list[0]; break; }
    for (int i : bl->h_list) bl->h_jitter[i] = base * std::pow(10.0, t);
    CKB(cudaMemcpyAsync(B.jitter, bl->h_jitter.data(), sizeof(double) * nl, cudaMemcpyHostToDevice, s));
    CKB(cudaMemcpyAsync(B.list, bl->h_list.data(), sizeof(int32_t) * bl->h_list.size(), cudaMemcpyHostToDevice, s));
    if (L.big) {
      launch_assemble(B.X, d, Ld, B.list, static_cast<int>(bl->h_list.size()), L.ld_max, B.jitter, B.Linv,
                      kernel, theta0.lengthscale, theta0.noise, theta0.outputscale, s);
      launch_big_chol_trtri(B.Linv, Ld, B.list, static_cast<int>(bl->h_list.size()), L.ld_max, B.status,
                            B.logdet_blk, B.u, B.bigscr, s);
    } else {
      launch_assemble(B.X, d, Ld, B.list, static_cast<int>(bl->h_list.size()), L.ld_max, B.jitter, B.Linv,
                      kernel, theta0.lengthscale, theta0.noise, theta0.outputscale, s);
      launch_chol_trtri(B.Linv, Ld, B.list, static_cast<int>(bl->h_list.size()), L.ld_max, B.status,
                        B.logdet_blk, B.u, s);
    }
    CKB(cudaGetLastError());
    CKB(cudaMemcpyAsync(hstat.data(), B.status, sizeof(int32_t) * nl, cudaMemcpyDeviceToHost, s));
    CKB(cudaStreamSynchronize(s));
  }
  for (double j : bl->h_jitter) bl->max_jitter = std::max(bl->max_jitter, j);
  if (shard) {
    // every rank learns the first failed block and the largest jitter (one host-level exchange)
    const double mine[2] = {static_cast<double>(fb + 1), bl->max_jitter};
    std::vector<double> all;
    nugpr_status xs_ = allgather_host(bl, mine, 2, all, s);
    if (xs_ != NUGPR_OK) { cudaStreamSynchronize(bas); delete bl; return xs_; }
    for (int r = 0; r < ctx->world; ++r) {
      const int f = static_cast<int>(all[2 * r]) - 1;
      if (f >= 0 && (fb < 0 || f < fb)) fb = f;
      bl->max_jitter = std::max(bl->max_jitter, all[2 * r + 1]);
    }
  }
  if (fb >= 0) {
    if (failed_block) *failed_block = fb;
    cudaStreamSynchronize(bas);           // the side stream still writes into the workspace
    delete bl;
    return fail(NUGPR_ERR_NOT_SPD, "cluster %d is not SPD after the jitter ladder", fb);
  }
  // H_i = Linv_i Linv_i^T ; logdet_R (K_rep, lambda_0, M were launched on the side stream)
  defer = defer && !ctx->prof;
  if (defer) {
    // deferred (nugpr_train): H on its own stream; the evaluations that read it wait on ev_h1
    if (!ctx->h_stream) CKB(cudaStreamCreateWithFlags(&ctx->h_stream, cudaStreamNonBlocking));
    if (!ctx->ev_h0) CKB(cudaEventCreateWithFlags(&ctx->ev_h0, cudaEventDisableTiming));
    if (!ctx->ev_h1) CKB(cudaEventCreateWithFlags(&ctx->ev_h1, cudaEventDisableTiming));
    CKB(cudaEventRecord(ctx->ev_h0, s));
    CKB(cudaStreamWaitEvent(ctx->h_stream, ctx->ev_h0, 0));
    launch_gemm_H(B.Linv, B.H, Ld, L.ld_max, !L.big, ctx->h_stream);
    CKB(cudaEventRecord(ctx->ev_h1, ctx->h_stream));
    bl->h_pending = true;
  } else {
    PROF(ctx, PC_GEMM, 0.0, s, launch_gemm_H(B.Linv, B.H, Ld, L.ld_max, !L.big, s));
  }
  if (shard) {
    // logdet_R = 2 sum_i sum_j log (R_i)_jj over ALL clusters: gather the per-cluster terms, then the
    // same fixed-order sum as one GPU
    double* lg = bl->E[0].xr;
    nugpr_status gs_ = gather_clusters(bl, B.logdet_blk, 1, lg, s);
    if (gs_ != NUGPR_OK) { cudaStreamSynchronize(bas); delete bl; return gs_; }
    launch_sum(lg, n_c, B.scal + 0, s);
  } else {
    launch_sum(B.logdet_blk, n_c, B.scal + 0, s);
  }
  CKB(cudaGetLastError());
  if (bas != s) CKB(cudaStreamWaitEvent(s, ctx->ev_aux[NUGPR_NUM_EVALS][1], 0));
  if (defer) {
    // no host read-back: logdet_R and lambda_0 stay on the device (the evaluations' records carry
    // them and check lambda_0 > 0 themselves)
    CKB(cudaGetLastError());
    bl->logdet_R = NAN;
    bl->lam0 = NAN;
    if (max_jitter) *max_jitter = bl->max_jitter;
    *out = bl;
    return NUGPR_OK;
  }
  double hs[2];
  int32_t lzi[3] = {0, 0, 0};
  CKB(cudaMemcpyAsync(hs, B.scal, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
  CKB(cudaMemcpyAsync(lzi, B.linfo, sizeof(int32_t) * 3, cudaMemcpyDeviceToHost, s));
  CKB(cudaStreamSynchronize(s));
#undef CKB
  prof_harvest(ctx);
  bl->logdet_R = hs[0];
  bl->lam0 = hs[1];
  if (max_jitter) *max_jitter = bl->max_jitter;
  if (!lzi[1]) {
    delete bl;
    return fail(NUGPR_ERR_INTERNAL, "lambda_0 Lanczos did not converge in %d iterations (n_c = %d)", lzi[0], n_c);
  }
  if (!(bl->lam0 > 0.0) || lzi[2]) {
    delete bl;
    return fail(NUGPR_ERR_DEGENERATE_REPS, "lambda_0 = %g is not certifiably > 0 (degenerate representatives)",
                hs[1]);
  }
  *out = bl;
  return NUGPR_OK;
}

extern "C" nugpr_status nugpr_blocks_destroy(nugpr_blocks* blocks) {
  delete blocks;
  return NUGPR_OK;
}

extern "C" nugpr_status nugpr_blocks_export(const nugpr_blocks* bl, int32_t what, void* dst, size_t bytes) {
  if (!bl || !dst) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  const HostLayout& L = bl->L;
  cudaStream_t s = bl->ctx->stream;
  CK(cudaSetDevice(bl->ctx->device));
  auto need = [&](size_t n) -> bool { return bytes >= n; };
  switch (what) {
    case 0:
    case 1: {
      size_t n = sizeof(double) * L.blk_total;
      if (!need(n)) return fail(NUGPR_ERR_INVALID_ARG, "need %zu bytes", n);
      if (what == 0 || L.big) {
        CK(cudaMemcpyAsync(dst, what == 0 ? bl->B.Linv : bl->B.H, n, cudaMemcpyDeviceToHost, s));
        break;
      }
      // H in the small layout is stored packed: expand to full ld_i x ld_i column-major blocks
      std::vector<double> pk(L.pk_total);
      CK(cudaMemcpyAsync(pk.data(), bl->B.H, sizeof(double) * L.pk_total, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      double* o = static_cast<double*>(dst);
      for (int i = 0; i < L.n_c; ++i) {
        const int ld = L.ld[i], mt = ld / 8;
        const double* bp = pk.data() + L.pboff[i];
        double* ob = o + L.boff[i];
        for (int c = 0; c < ld; ++c)
          for (int r = 0; r < ld; ++r) {
            const int rr = std::max(r, c), cc = std::min(r, c);
            const int I = rr / 8, K = cc / 8;
            ob[static_cast<int64_t>(c) * ld + r] = bp[static_cast<int64_t>(pk_tile(I, K, mt)) * 64 + swz(rr % 8, cc % 8)];
          }
      }
      return NUGPR_OK;
    }
    case 2: {
      size_t n = sizeof(double) * L.n;
      if (!need(n)) return fail(NUGPR_ERR_INVALID_ARG, "need %zu bytes", n);
      std::vector<double> up(L.n_pad);
      CK(cudaMemcpyAsync(up.data(), bl->B.u, sizeof(double) * L.n_pad, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      double* o = static_cast<double*>(dst);
      for (int i = 0; i < L.n_c; ++i)
        for (int64_t r = 0; r < L.off[i + 1] - L.off[i]; ++r) o[L.off[i] + r] = up[L.poff[i] + r];
      return NUGPR_OK;
    }
    case 3: {
      size_t n = sizeof(double) * L.n_c;
      if (!need(n)) return fail(NUGPR_ERR_INVALID_ARG, "need %zu bytes", n);
      CK(cudaMemcpyAsync(dst, bl->B.jitter, n, cudaMemcpyDeviceToHost, s));
      break;
    }
    case 4: {
      if (!need(2 * sizeof(double))) return fail(NUGPR_ERR_INVALID_ARG, "need 16 bytes");
      CK(cudaMemcpyAsync(dst, bl->B.scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
      break;
    }
    case 5: {
      size_t n = sizeof(double) * bl->n_cg * bl->n_cg;
      if (!need(n)) return fail(NUGPR_ERR_INVALID_ARG, "need %zu bytes", n);
      CK(cudaMemcpyAsync(dst, bl->B.M, n, cudaMemcpyDeviceToHost, s));
      break;
    }
    case 6: {
      size_t n = sizeof(int32_t) * L.n_c;
      if (!need(n)) return fail(NUGPR_ERR_INVALID_ARG, "need %zu bytes", n);
      memcpy(dst, L.ld.data(), n);
      return NUGPR_OK;
    }
    case 7: {
      size_t n = sizeof(double) * bl->last_m * L.n;
      if (bl->last_m == 0 || !need(n)) return fail(NUGPR_ERR_INVALID_ARG, "no probes / need %zu bytes", n);
      launch_probe_gen(bl->last_seed, bl->last_m, L.n, bl->B.Zexport, s);
      CKL();
      CK(cudaMemcpyAsync(dst, bl->B.Zexport, n, cudaMemcpyDeviceToHost, s));
      break;
    }
    case 8:
    case 9: {   // Lanczos {iterations, converged}: 8 = the build's, 9 = slot 0's last generic eval
      if (!need(2 * sizeof(int32_t))) return fail(NUGPR_ERR_INVALID_ARG, "need 8 bytes");
      CK(cudaMemcpyAsync(dst, what == 8 ? bl->B.linfo : bl->E[0].linfo, 2 * sizeof(int32_t),
                         cudaMemcpyDeviceToHost, s));
      break;
    }
    default:
      return fail(NUGPR_ERR_INVALID_ARG, "unknown export %d", what);
  }
  CK(cudaStreamSynchronize(s));
  return NUGPR_OK;
}

// ------------------------------------------------------------------------------------------
// Row A0: clustering (cluster_kernels.cu).  Host code only sequences the Lloyd iterations
// (one 4-byte "changed" read-back per iteration) and draws the Forgy row indices.
namespace {
struct KmWs {
  double *X, *C, *C0, *Xs, *yin, *ys, *score;
  unsigned long long *S, *cnt, *amax;
  int32_t *a0, *a1, *changed;
  long long* hist;
  int64_t *perm, *off, *med, *idx;
};
size_t km_carve(Carver& c, int64_t n, int d, int n_c, KmWs& w) {
  const int64_t nch = km_chunks(n);
  w.X = c.take<double>(static_cast<size_t>(n) * d);
  w.Xs = c.take<double>(static_cast<size_t>(n) * d);
  w.yin = c.take<double>(n);
  w.ys = c.take<double>(n);
  w.score = c.take<double>(n);
  w.C = c.take<double>(static_cast<size_t>(n_c) * d);
  w.C0 = c.take<double>(static_cast<size_t>(n_c) * d);
  w.S = c.take<unsigned long long>(static_cast<size_t>(n_c) * d);
  w.cnt = c.take<unsigned long long>(n_c);
  w.amax = c.take<unsigned long long>(1);
  w.a0 = c.take<int32_t>(n);
  w.a1 = c.take<int32_t>(n);
  w.changed = c.take<int32_t>(1);
  w.hist = c.take<long long>(static_cast<size_t>(nch) * n_c);
  w.perm = c.take<int64_t>(n);
  w.off = c.take<int64_t>(n_c + 1);
  w.med = c.take<int64_t>(n_c);
  w.idx = c.take<int64_t>(n_c);
  return c.pos + 256;
}
}  // namespace

extern "C" nugpr_status nugpr_cluster_workspace_size(int64_t n, int32_t d, int32_t n_c, size_t* bytes) {
  if (!bytes) return fail(NUGPR_ERR_INVALID_ARG, "bytes is NULL");
  if (n < 1 || d < 1 || d > 32 || n_c < 1 || n_c > n) return fail(NUGPR_ERR_INVALID_ARG, "need n >= n_c >= 1, 1 <= d <= 32");
  Carver c(nullptr);
  KmWs w;
  *bytes = km_carve(c, n, d, n_c, w);
  return NUGPR_OK;
}

extern "C" nugpr_status nugpr_cluster(nugpr_ctx* ctx, const double* X, int64_t n, int32_t d, int32_t n_c,
                                      const double* init_centers, uint64_t seed, int32_t max_iter,
                                      int32_t rep_mode, int32_t kernel, nugpr_theta theta, const double* y,
                                      void* workspace, size_t ws_bytes, int64_t* perm, int64_t* offsets,
                                      double* reps, double* X_sorted, double* y_sorted, int32_t* iters) {
  if (!ctx || !X || !workspace || !offsets) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  size_t need = 0;
  RET(nugpr_cluster_workspace_size(n, d, n_c, &need));
  if (ws_bytes < need) return fail(NUGPR_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return fail(NUGPR_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  if (max_iter < 0) return fail(NUGPR_ERR_INVALID_ARG, "max_iter < 0");
  if (rep_mode < NUGPR_REP_GIVEN || rep_mode > NUGPR_REP_MEDOID) return fail(NUGPR_ERR_INVALID_ARG, "bad rep_mode");
  if (rep_mode == NUGPR_REP_MEDOID && (kernel < 0 || kernel > 2 || !theta_ok(theta)))
    return fail(NUGPR_ERR_INVALID_ARG, "MEDOID needs a valid kernel and theta");
  CK(cudaSetDevice(ctx->device));
  cudaGetLastError();
  cudaStream_t s = ctx->stream;
  Carver c(workspace);
  KmWs w;
  km_carve(c, n, d, n_c, w);
  const size_t xb = sizeof(double) * static_cast<size_t>(n) * d, cb = sizeof(double) * static_cast<size_t>(n_c) * d;
  CK(cudaMemcpyAsync(w.X, X, xb, cudaMemcpyDefault, s));
  if (init_centers) {
    CK(cudaMemcpyAsync(w.C0, init_centers, cb, cudaMemcpyDefault, s));
  } else {
    // Forgy: candidate t of centre j = splitmix64_seed((j << 32) | t) mod n, first one not taken
    std::vector<int64_t> idx(n_c);
    std::vector<char> taken(static_cast<size_t>(n), 0);
    for (int j = 0; j < n_c; ++j) {
      for (uint64_t t = 0;; ++t) {
        const int64_t i = static_cast<int64_t>(splitmix64_at(seed, (static_cast<uint64_t>(j) << 32) | t) %
                                               static_cast<uint64_t>(n));
        if (!taken[i]) { taken[i] = 1; idx[j] = i; break; }
      }
    }
    CK(cudaMemcpyAsync(w.idx, idx.data(), sizeof(int64_t) * n_c, cudaMemcpyHostToDevice, s));
    launch_km_gather(w.X, d, w.idx, nullptr, n_c, w.C0, s);
  }
  CK(cudaMemcpyAsync(w.C, w.C0, cb, cudaMemcpyDeviceToDevice, s));
  // fixed-point scale 2^s, s = 62 - ceil(log2(max|x| n))
  CK(cudaMemsetAsync(w.amax, 0, sizeof(unsigned long long), s));
  launch_km_absmax(w.X, static_cast<int64_t>(n) * d, w.amax, s);
  unsigned long long amax_bits = 0;
  CK(cudaMemcpyAsync(&amax_bits, w.amax, sizeof(amax_bits), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  double amax;
  memcpy(&amax, &amax_bits, sizeof(double));
  const int shift = (amax == 0.0) ? 62 : static_cast<int>(62 - std::ceil(std::log2(amax * static_cast<double>(n))));
  const double scale = std::ldexp(1.0, shift), inv_scale = std::ldexp(1.0, -shift);
  CK(cudaMemsetAsync(w.S, 0, sizeof(unsigned long long) * static_cast<size_t>(n_c) * d, s));
  CK(cudaMemsetAsync(w.cnt, 0, sizeof(unsigned long long) * n_c, s));
  // Lloyd: assign; repeat {update; assign} until no change or max_iter updates
  int32_t* a_cur = w.a0;
  int32_t* a_nxt = w.a1;
  launch_km_assign(w.X, n, d, n_c, w.C, nullptr, a_cur, scale, w.S, w.cnt, w.changed, s);
  CKL();
  int it = 0;
  while (it < max_iter) {
    launch_km_update(n_c, d, inv_scale, w.S, w.cnt, w.C, s);
    ++it;
    CK(cudaMemsetAsync(w.changed, 0, sizeof(int32_t), s));
    launch_km_assign(w.X, n, d, n_c, w.C, a_cur, a_nxt, scale, w.S, w.cnt, w.changed, s);
    CKL();
    std::swap(a_cur, a_nxt);
    CK(cudaMemcpyAsync(ctx->h_flag, w.changed, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!*ctx->h_flag) break;
  }
  if (iters) *iters = it;
  // stable counting sort by (cluster, original index)
  launch_km_sort(a_cur, n, n_c, w.hist, w.perm, w.off, s);
  CKL();
  CK(cudaMemcpyAsync(offsets, w.off, sizeof(int64_t) * (n_c + 1), cudaMemcpyDeviceToHost, s));
  launch_km_gather(w.X, d, w.perm, nullptr, n, w.Xs, s);
  if (y) {
    CK(cudaMemcpyAsync(w.yin, y, sizeof(double) * n, cudaMemcpyDefault, s));
    launch_km_gather(w.yin, 1, w.perm, nullptr, n, w.ys, s);
  }
  CKL();
  CK(cudaStreamSynchronize(s));
  int64_t bmax = 0;
  bool empty = false;
  for (int j = 0; j < n_c; ++j) {
    bmax = std::max<int64_t>(bmax, offsets[j + 1] - offsets[j]);
    if (offsets[j + 1] == offsets[j]) empty = true;
  }
  if (reps) {
    if (rep_mode == NUGPR_REP_GIVEN) {
      CK(cudaMemcpyAsync(reps, w.C0, cb, cudaMemcpyDefault, s));
    } else if (rep_mode == NUGPR_REP_CENTROID) {
      CK(cudaMemcpyAsync(reps, w.C, cb, cudaMemcpyDefault, s));
    } else {
      if (empty) return fail(NUGPR_ERR_SHAPE, "MEDOID representatives need non-empty clusters");
      launch_km_medoids(w.Xs, d, w.off, n_c, bmax, kernel, theta.lengthscale, theta.outputscale, w.score, w.med, s);
      launch_km_gather(w.Xs, d, w.med, nullptr, n_c, w.C0, s);
      CKL();
      CK(cudaMemcpyAsync(reps, w.C0, cb, cudaMemcpyDefault, s));
    }
  }
  if (perm) CK(cudaMemcpyAsync(perm, w.perm, sizeof(int64_t) * n, cudaMemcpyDefault, s));
  if (X_sorted) CK(cudaMemcpyAsync(X_sorted, w.Xs, xb, cudaMemcpyDefault, s));
  if (y_sorted && y) CK(cudaMemcpyAsync(y_sorted, w.ys, sizeof(double) * n, cudaMemcpyDefault, s));
  CK(cudaStreamSynchronize(s));
  if (empty) return fail(NUGPR_ERR_SHAPE, "a cluster is empty after k-means");
  return NUGPR_OK;
}

// ------------------------------------------------------------------------------------------
// One evaluation = host-side parameter setup and mode-specific pre-work (Eq. 23-28), the CG
// solves (rows A4-A5) and the trace / final kernels (A5-A7).  In graph mode the CG loop and the
// tail are ONE CUDA graph per (workspace, slot): a conditional WHILE node whose condition the
// update kernel's last CTA sets on the device, so an evaluation needs no host round trip and
// every operator mode shares the graph (mode data live in the device EvalParams).  With
// profiling on (bench.py's roofline pass) the same kernels are launched directly, serialised,
// with CUDA events around each one.

struct IterArgs {
  ApplyArgs a1, a2, a3, a4;
  LowrankArgs t1, t2, t3, t4;   // big-block layout only: T = M'S before each apply
  UpdateArgs ua;
  int ncp = 0;
  bool lowrank = false;         // separate low-rank launches (big-block layout)
  int ncol = 0;
  bool mbcg = false;            // NEXT-4: one apply per iteration (CG on A for every column)
};

// Launch arguments of one evaluation's CG iteration and trace tail (slot e, ncol RHS columns).
//  apply 1: V = A p with p = r + beta p fused (P_new written), epilogue S(V)
//  apply 2: q = A V + 4 V + p (probe columns: Q(A) p), q = V (y column); dots p^T q -> alpha
//  update : x += alpha p, r -= alpha q; r^T r and S(r) -> beta, freezing, the graph's while condition
//  trace  : V = A x (S(V)), U = 3 A V - 3 x (probe columns: P(A) x, Eq. 10) / x (y column), dotted with
//           the right-hand sides -> t_j and quad (FIN_TRACE)
// The packed apply forms the low-rank rows M'S(D) itself from the S rows its input's producer wrote
// (S_D); the big-block layout keeps a lowrank_kernel launch before each apply.
static nugpr_status make_iter_args(nugpr_blocks* bl, EvalDev& e, int ncol, IterArgs& A, bool mbcg = false) {
  const HostLayout& L = bl->L;
  const LayoutDev& Ld = bl->Ld;
  const BlocksDev& B = bl->B;
  A.ncp = (ncol + 1) & ~1;
  A.ncol = ncol;
  A.lowrank = L.big;
  ApplyArgs& a1 = A.a1;
  memset(&a1, 0, sizeof(a1));
  a1.L = Ld; a1.prm = e.prm; a1.st = e.st; a1.u = B.u; a1.jitter = B.jitter; a1.ncol = ncol;
  a1.Pbuf[0] = e.Pb[0]; a1.Pbuf[1] = e.Pb[1]; a1.SPbuf[0] = e.SPb[0]; a1.SPbuf[1] = e.SPb[1];
  a1.alpha_hist = e.ah; a1.hist_stride = HIST;
  a1.ld_max = L.ld_max;
  a1.lr_row0 = 0; a1.lr_nc = L.n_c;
  a1.Tbuf = e.Tbuf;
  a1.split_part = e.split; a1.split_ticket = e.split_tick;
  if (L.big) {
    a1.big = 1;
    a1.grid = Ld.n_tiles;
  } else {
    if (!plan_packed_apply(L.ld_max, ncol, bl->f32, L.seg_max, bl->n_cg, a1))
      return fail(NUGPR_ERR_SHAPE, "packed apply does not fit shared memory (ld_max=%d, ncol=%d, pieces/CTA=%d)",
                  L.ld_max, ncol, L.seg_max);
    a1.grid = Ld.n_seg_ctas;
  }
  ApplyArgs& a2 = A.a2;
  a2 = a1;
  a1.D = e.R; a1.S_D = e.SR; a1.fuse_p = 1; a1.out = e.V; a1.epi = EPI_S; a1.Sout = e.SV;
  a1.fin = FIN_NONE; a1.gate = 1;
  for (int c = 0; c < MAXC; ++c) { a1.cA[c] = 1.0; a1.cV[c] = 0.0; a1.cP[c] = 0.0; }
  a2.D = e.V; a2.S_D = e.SV; a2.fuse_p = 0; a2.out = e.Q; a2.use_par_p2 = 1; a2.epi = EPI_DOT;
  a2.dots = e.dots; a2.fin = FIN_ALPHA; a2.gate = 1;
  for (int c = 0; c < MAXC; ++c) {
    if (c == 0) { a2.cA[c] = 0.0; a2.cV[c] = 1.0; a2.cP[c] = 0.0; }
    else { a2.cA[c] = 1.0; a2.cV[c] = 4.0; a2.cP[c] = 1.0; }
  }
  UpdateArgs& ua = A.ua;
  memset(&ua, 0, sizeof(ua));
  ua.L = Ld; ua.prm = e.prm; ua.st = e.st; ua.u = B.u; ua.X = e.X; ua.R = e.R; ua.Q = e.Q;
  ua.Pbuf[0] = e.Pb[0]; ua.Pbuf[1] = e.Pb[1]; ua.rr_part = e.rrp; ua.SR_part = e.SR;
  ua.SPbuf[0] = e.SPb[0]; ua.SPbuf[1] = e.SPb[1];
  ua.beta_hist = e.bh; ua.hist_stride = HIST; ua.ncol = ncol; ua.cond = 0;
  ApplyArgs& a3 = A.a3;
  a3 = a1;
  a3.D = e.X; a3.S_D = e.SX; a3.fuse_p = 0; a3.out = e.V; a3.epi = EPI_S; a3.Sout = e.SV;
  a3.fin = FIN_NONE; a3.gate = 0; a3.use_par_p2 = 0; a3.P2 = nullptr;
  ApplyArgs& a4 = A.a4;
  a4 = a3;
  a4.D = e.V; a4.S_D = e.SV; a4.out = e.U; a4.P2 = e.X; a4.epi = EPI_DOT; a4.Y2 = e.RHS; a4.dots = e.dots;
  a4.fin = FIN_TRACE;
  for (int c = 0; c < MAXC; ++c) {
    if (c == 0) { a4.cA[c] = 0.0; a4.cV[c] = 0.0; a4.cP[c] = 1.0; }
    else { a4.cA[c] = 3.0; a4.cV[c] = 0.0; a4.cP[c] = -3.0; }
  }
  if (mbcg) {
    // NEXT-4 (mBCG on A): apply 1 alone per iteration, q = A p for every column, its dots with the
    // freshly formed p (Y2 := D = P_new) -> alpha; no Q(A) second apply, no Pade tail
    A.mbcg = true;
    a1.out = e.Q; a1.epi = EPI_DOT; a1.Sout = nullptr; a1.use_par_p2 = 2; a1.P2 = nullptr;
    a1.dots = e.dots; a1.fin = FIN_ALPHA;
  }
  // big-block layout: separate low-rank launches, S partials per 64-row tile (summed via tile0)
  LowrankArgs& t1 = A.t1;
  memset(&t1, 0, sizeof(t1));
  t1.task0 = L.big ? B.tile0 : nullptr;
  t1.st = e.st; t1.prm = e.prm; t1.Mp = nullptr; t1.S = e.SR; t1.SPbuf[0] = e.SPb[0]; t1.SPbuf[1] = e.SPb[1];
  t1.fuse_p = 1; t1.T = e.Tbuf; t1.n_c = L.n_c; t1.ncol = ncol; t1.gate = 1;
  t1.row0 = 0; t1.nrows = L.n_c;
  A.t2 = t1; A.t2.S = e.SV; A.t2.fuse_p = 0;
  A.t3 = A.t2; A.t3.S = e.SX; A.t3.gate = 0;
  A.t4 = A.t2; A.t4.S = e.SV; A.t4.gate = 0;
  if (bl->shard) {
    // PAR-2: the partials of this rank's clusters go to their global slots of the zero-padded send
    // array xs = [rr | S(r) | S(A p), p^T q, S(x), trace dots] ([3][n_cg][MAXC]); the exchange fills
    // xr with every rank's; finalisers run as fin_kernel after it; the apply reads the GLOBAL S rows
    // and forms M'S for its local rows only (lr_row0 = c_lo)
    if (mbcg || L.big)
      return fail(NUGPR_ERR_UNSUPPORTED, "cluster sharding: mBCG / big blocks not supported");
    const size_t G = static_cast<size_t>(bl->n_cg) * MAXC, o = static_cast<size_t>(bl->c_lo) * MAXC;
    a1.Sout = e.xs + 2 * G + o;
    a2.dots = e.xs + 2 * G + o; a2.fin = FIN_NONE;
    a3.Sout = e.xs + 2 * G + o;
    a4.dots = e.xs + 2 * G + o; a4.fin = FIN_NONE;
    ua.rr_part = e.xs + o; ua.SR_part = e.xs + G + o; ua.nofin = 1;
    a1.S_D = e.xr + G;
    a2.S_D = e.xr + 2 * G;
    a3.S_D = e.xr + 2 * G;
    a4.S_D = e.xr + 2 * G;
    for (ApplyArgs* x : {&a1, &a2, &a3, &a4}) { x->lr_row0 = bl->c_lo; x->lr_nc = bl->n_cg; }
  }
  return NUGPR_OK;
}

// Direct launches of one CG iteration / the trace tail.
static void launch_iteration(const IterArgs& A, cudaStream_t s) {
  if (A.lowrank) launch_lowrank(A.t1, A.ncp, s);
  launch_apply(A.a1, A.ncp, s);
  if (A.mbcg) { launch_update(A.ua, A.ncp, s); return; }
  if (A.lowrank) launch_lowrank(A.t2, A.ncp, s);
  launch_apply(A.a2, A.ncp, s);
  launch_update(A.ua, A.ncp, s);
}
static void launch_tail(nugpr_blocks* bl, EvalDev& e, const IterArgs& A, int ncol, cudaStream_t s) {
  launch_spart(bl->Ld, bl->B.u, e.X, ncol, e.SX, s);
  if (A.lowrank) launch_lowrank(A.t3, A.ncp, s);
  launch_apply(A.a3, A.ncp, s);
  if (A.lowrank) launch_lowrank(A.t4, A.ncp, s);
  launch_apply(A.a4, A.ncp, s);
}

static int quad_nparts(const nugpr_blocks* bl) {
  return quad_parts(bl->L.n_pad, static_cast<int>(bl->Ld.n_tiles) * MAXC);
}
static void launch_tail_final(nugpr_blocks* bl, EvalDev& e, const IterArgs& A, int ncol, int logdet_mode,
                              cudaStream_t s) {
  if (A.mbcg) {
    const int np = quad_nparts(bl);
    launch_quad_part(e.RHS, e.X, bl->L.n_pad, np, e.SX, s);
    launch_final(e.st, e.prm, e.ah, e.bh, HIST, e.slqw, bl->B.scal + 0, static_cast<double>(bl->L.n), ncol,
                 logdet_mode, e.out, s, e.SX, np);
    return;
  }
  launch_tail(bl, e, A, ncol, s);
  launch_final(e.st, e.prm, e.ah, e.bh, HIST, e.slqw, bl->B.scal + 0, static_cast<double>(bl->L.n),
               ncol, logdet_mode, e.out, s);
}

// PAR-2 (sharded) CG iteration / tail: the same kernels on this rank's clusters with the three
// partial exchanges per iteration and the finalisers as fin_kernel launches after them; enqueued
// directly (host-driven loop) or captured into the evaluation graph when the exchanges are the
// library's own NCCL collectives (cond: the graph's while handle, set by FIN_UPDATE).
static nugpr_status launch_iteration_shard(nugpr_ctx* ctx, nugpr_blocks* bl, EvalDev& e, const IterArgs& A,
                                           int ncol, cudaStream_t s, unsigned long long cond, double apply_bytes = 0.0) {
  const size_t XG = static_cast<size_t>(bl->n_cg) * MAXC;
  double* xs = e.xs, *xr = e.xr;
  const int cls = PC_APPLY_B;
  PROF(ctx, cls, apply_bytes, s, launch_apply(A.a1, A.ncp, s));
  RET(xchg(ctx, xs + 2 * XG, xr + 2 * XG, XG, s));                        // S(A p)
  PROF(ctx, cls, apply_bytes, s, launch_apply(A.a2, A.ncp, s));
  RET(xchg(ctx, xs + 2 * XG, xr + 2 * XG, XG, s));                        // p^T q
  launch_fin(FIN_ALPHA, e.st, e.prm, xr + 2 * XG, bl->n_cg, ncol, e.ah, HIST, s);
  PROF(ctx, PC_UPDATE, 0.0, s, launch_update(A.ua, A.ncp, s));
  RET(xchg(ctx, xs, xr, 2 * XG, s));                                      // r^T r, S(r)
  launch_fin(FIN_UPDATE, e.st, e.prm, xr, bl->n_cg, ncol, e.bh, HIST, s, xr + XG, e.SPb[0], e.SPb[1], cond);
  return NUGPR_OK;
}
static nugpr_status launch_tail_shard(nugpr_ctx* ctx, nugpr_blocks* bl, EvalDev& e, const IterArgs& A, int ncol,
                                      int logdet_mode, cudaStream_t s, double apply_bytes = 0.0) {
  const size_t XG = static_cast<size_t>(bl->n_cg) * MAXC, XO = static_cast<size_t>(bl->c_lo) * MAXC;
  double* xs = e.xs, *xr = e.xr;
  launch_spart(bl->Ld, bl->B.u, e.X, ncol, xs + 2 * XG + XO, s);
  RET(xchg(ctx, xs + 2 * XG, xr + 2 * XG, XG, s));                        // S(x)
  PROF(ctx, PC_APPLY_B, apply_bytes, s, launch_apply(A.a3, A.ncp, s));
  RET(xchg(ctx, xs + 2 * XG, xr + 2 * XG, XG, s));                        // S(A x)
  PROF(ctx, PC_APPLY_B, apply_bytes, s, launch_apply(A.a4, A.ncp, s));
  RET(xchg(ctx, xs + 2 * XG, xr + 2 * XG, XG, s));                        // quad, trace dots
  launch_fin(FIN_TRACE, e.st, e.prm, xr + 2 * XG, bl->n_cg, ncol, nullptr, HIST, s);
  launch_final(e.st, e.prm, e.ah, e.bh, HIST, e.slqw, bl->B.scal + 0, static_cast<double>(bl->n_glob),
               ncol, logdet_mode, e.out, s);
  CKL();
  return NUGPR_OK;
}

// Graph of one slot: while (any column active) { CG iteration }; spart; trace applies; final.
static std::string graph_key(const nugpr_blocks* bl, int slot, int ncol, int logdet_mode) {
  char buf[160];
  const HostLayout& L = bl->L;
  uint64_t h = 1469598103934665603ull;    // FNV-1a over the offsets (pointers follow from them)
  for (int64_t v : L.off) { h ^= static_cast<uint64_t>(v); h *= 1099511628211ull; }
  snprintf(buf, sizeof(buf), "%p|%zu|%d|%d|%d|%d|%llx|%d|%d", static_cast<const void*>(bl->ws_base), bl->E.size(),
           slot, ncol, logdet_mode, L.d, static_cast<unsigned long long>(h), L.n_c, bl->f32 ? 1 : 0);
  return std::string(buf);
}

static nugpr_status get_graph(nugpr_ctx* ctx, nugpr_blocks* bl, int slot, int ncol, int logdet_mode,
                              cudaGraphExec_t* out);

// Enqueue one evaluation on stream s with slot e; the record lands in e.out (device).  `limit`
// receives the host-known iteration bound (replay) for the launch accounting.
static nugpr_status enqueue_eval(nugpr_ctx* ctx, nugpr_blocks* bl, int slot, const double* y_dev,
                                 nugpr_theta th, const nugpr_solve_cfg* cfg, cudaStream_t s, int* mode_out,
                                 EvalParams* hstage, bool prep_only = false) {
  EvalDev& e = bl->E[slot];
  const HostLayout& L = bl->L;
  const LayoutDev& Ld = bl->Ld;
  const BlocksDev& B = bl->B;
  const nugpr_theta t0 = bl->theta0;
  const int m = cfg->num_probes;
  const int ncol = 1 + m;
  const int max_iter = cfg->cg_max_iter;
  EvalParams& P = *hstage;                  // pinned host staging (async upload below)
  memset(&P, 0, sizeof(P));
  P.tol = cfg->cg_tol;
  P.max_iter = max_iter;
  P.ncol = ncol;
  P.mscale = 1.0;
  P.Mp = B.M;
  if (cfg->replay_iters) {
    P.replay = 1;
    for (int c = 0; c < ncol; ++c) P.replay_iters[c] = std::min(cfg->replay_iters[c], max_iter);
  }
  const double* lam0_ptr = B.scal + 1;
  int mode;
  const bool same_l = th.lengthscale == t0.lengthscale, same_s = th.noise == t0.noise,
             same_a = th.outputscale == t0.outputscale;
  if (same_l && same_s && same_a) {                       // Eq. (23)
    mode = NUGPR_MODE_BASELINE;
    P.a = 1.0; P.B = nullptr;
  } else if (same_l && same_a) {                          // Eq. (24)
    mode = NUGPR_MODE_NOISE;
    P.a = 1.0; P.b0 = th.noise - t0.noise; P.b1 = 0.0; P.B = B.H;
  } else if (same_l && same_s) {                          // Eq. (25)
    mode = NUGPR_MODE_SCALE;
    const double r = (th.outputscale - t0.outputscale) / t0.outputscale;
    P.a = 1.0 + r; P.b0 = -t0.noise * r; P.b1 = -r; P.B = B.H; P.mscale = 1.0 + r;
  } else {                                                // generic (lengthscale step)
    mode = NUGPR_MODE_GENERIC;
    P.a = 0.0; P.b0 = 1.0; P.b1 = 0.0; P.B = e.G; P.Mp = e.M;
    // K_rep(theta') and its lambda_0 (latency-bound Lanczos) run on a side stream while this
    // stream assembles K_i(lambda') and forms G (FP64 tensor-pipe GEMMs)
    RET(ensure_aux(ctx, slot));
    cudaStream_t as = ctx->prof ? s : ctx->aux_stream[slot];
    if (as != s) {
      CK(cudaEventRecord(ctx->ev_aux[slot][0], s));
      CK(cudaStreamWaitEvent(as, ctx->ev_aux[slot][0], 0));
    }
    launch_krep(B.reps, bl->n_cg, L.d, bl->kind, th.lengthscale, th.outputscale, e.Krep, as);
    CKL();
    nugpr_status ls;
    PROF(ctx, PC_LANCZOS, 0.0, as, ls = enqueue_lambda0(bl, e.Krep, B.v0, e.lz, e.scal, e.v0, e.M, e.linfo, as));
    RET(ls);
    if (as != s) CK(cudaEventRecord(ctx->ev_aux[slot][1], as));
    PROF(ctx, PC_OTHER, 0.0, s,
         launch_assemble(B.X, L.d, Ld, nullptr, 0, L.ld_max, B.jitter, e.G, bl->kind, th.lengthscale,
                         th.noise, th.outputscale, s));
    PROF(ctx, PC_GEMM, 0.0, s, launch_gemm_KLt(e.G, B.Linv, e.T, Ld, L.ld_max, s));
    PROF(ctx, PC_GEMM, 0.0, s, launch_gemm_LT(B.Linv, e.T, e.G, Ld, L.ld_max, !L.big, s));
    CKL();
    if (as != s) CK(cudaStreamWaitEvent(s, ctx->ev_aux[slot][1], 0));
    lam0_ptr = e.scal;
  }
  if (P.B == B.H && bl->h_pending) CK(cudaStreamWaitEvent(s, ctx->ev_h1, 0));   // deferred build's H
  bl->f32 = cfg->block_storage == NUGPR_BLOCKS_F32;
  if (bl->f32) {
    if (L.big) return fail(NUGPR_ERR_UNSUPPORTED, "FP32 block storage needs clusters <= %d points", LD_SMALL_MAX);
    if (mode == NUGPR_MODE_GENERIC) {
      float* g32 = reinterpret_cast<float*>(e.T);            // free after the G GEMMs
      launch_d2f(e.G, g32, L.pk_total, s);
      P.B32 = g32;
    } else if (P.B) {
      if (!bl->h32_ready) { launch_d2f(B.H, B.H32, L.pk_total, s); bl->h32_ready = true; }
      P.B32 = B.H32;
    }
    CKL();
  }
  P.mode = mode;
  P.lam0_src = lam0_ptr;
  P.lam0_mul = 1.0;
  P.lz_info = (mode == NUGPR_MODE_GENERIC) ? e.linfo : B.linfo;
  if (mode_out) *mode_out = mode;
  if (mode == NUGPR_MODE_SCALE) {
    // lam0(theta') = (1+r) lam0(theta0): one scalar, computed on the host from the value the
    // build read back (reported in the record only)
    // (read on the device from the build's lambda_0: the build need not sync to the host first)
    P.lam0_src = B.scal + 1;
    P.lam0_mul = P.mscale;
  }
  CK(cudaMemcpyAsync(e.prm, &P, sizeof(P), cudaMemcpyHostToDevice, s));
  // the workspace is caller memory with arbitrary contents: the CG state (incl. the
  // self-resetting last-CTA tickets) and the S partials start from zero every evaluation
  CK(cudaMemsetAsync(e.st, 0, sizeof(CGState), s));
  // rhs + init
  const size_t XG = static_cast<size_t>(bl->n_cg) * MAXC, XO = static_cast<size_t>(bl->c_lo) * MAXC;
  if (bl->shard) CK(cudaMemsetAsync(e.xs, 0, sizeof(double) * 3 * XG, s));   // zero padding of the exchanges
  RhsArgs ra;
  ra.L = Ld; ra.prm = e.prm; ra.st = e.st; ra.Linv = B.Linv; ra.y = y_dev + bl->pos0;
  ra.probes = cfg->probes; ra.seed = cfg->probe_seed; ra.u = B.u; ra.RHS = e.RHS; ra.R = e.R;
  ra.X = e.X; ra.P0 = e.Pb[0]; ra.SP0 = e.SPb[0]; ra.SR_part = e.SR; ra.rr_part = e.rrp; ra.ncol = ncol;
  ra.cy = bl->cy_ready ? B.cy : nullptr;
  ra.cy_out = nullptr;
  ra.pos0 = bl->pos0; ra.n_glob = bl->n_glob; ra.nofin = 0;
  if (bl->shard) {
    ra.rr_part = e.xs + XO; ra.SR_part = e.xs + XG + XO; ra.SP0 = e.xs + 2 * XG + XO; ra.nofin = 1;
  }
  PROF(ctx, PC_RHS, 0.0, s, launch_rhs_init(ra, L.ld_max, s));
  CKL();
  if (bl->shard) {
    // PAR-2: r^T r and S(r) of every rank -> CG state; S(p_0) = S(r_0) (global)
    RET(xchg(ctx, e.xs, e.xr, 2 * XG, s));
    launch_fin(FIN_INIT, e.st, e.prm, e.xr, bl->n_cg, ncol, nullptr, HIST, s);
    CK(cudaMemcpyAsync(e.SPb[0], e.xr + XG, sizeof(double) * XG, cudaMemcpyDeviceToDevice, s));
    CKL();
  }
  if (prep_only) return NUGPR_OK;
  const bool useB = P.B != nullptr;
  if (!ctx->prof && ctx->use_graphs && (!bl->shard || (ctx->nccl && ctx->shard_graph_ok))) {
    cudaGraphExec_t ex = nullptr;
    const nugpr_status gs = get_graph(ctx, bl, slot, ncol, cfg->logdet_mode, &ex);
    if (gs == NUGPR_OK) {
      CK(cudaGraphLaunch(ex, s));
      return NUGPR_OK;
    }
    if (!bl->shard) return gs;
    // the NCCL collectives could not be captured into a conditional graph on this system: keep the
    // host-driven sharded loop (same kernels, same exchanges)
    cudaGetLastError();
    ctx->shard_graph_ok = false;
  }
  // direct launches (profiling / NUGPR_OPT_GRAPHS = 0): host polls the activity flag every CH iterations
  IterArgs A;
  RET(make_iter_args(bl, e, ncol, A, cfg->logdet_mode == NUGPR_LOGDET_MBCG));
  // algorithmic bytes of one apply: w (P + 2 n c + n + n_c^2) with P = sum b_i (b_i + 1) / 2
  // for the packed symmetric blocks of the small layout, sum b_i^2 for the full blocks of the big one
  double sum_p = 0.0;
  for (int i = 0; i < L.n_c; ++i) {
    const double b = static_cast<double>(L.off[i + 1] - L.off[i]);
    sum_p += L.big ? b * b : 0.5 * b * (b + 1.0);
  }
  const double vec_bytes = 8.0 * (2.0 * L.n * ncol + L.n + static_cast<double>(L.n_c) * L.n_c);
  const double apply_bytes = (useB ? (bl->f32 ? 4.0 : 8.0) * sum_p : 0.0) + vec_bytes;   // B as stored
  const int apply_cls = useB ? PC_APPLY_B : PC_APPLY_LR;
  const int limit = cfg->replay_iters ? [&] { int mx = 0; for (int c = 0; c < ncol; ++c) mx = std::max(mx, P.replay_iters[c]); return mx; }()
                                      : max_iter;
  const int CH = 4;
  int done = 0;
  if (bl->shard) {
    // PAR-2 CG (callback exchanges or profiling): host-driven, the activity flag read every CH iterations
    while (done < limit) {
      for (int q = 0; q < CH && done < limit; ++q, ++done)
        RET(launch_iteration_shard(ctx, bl, e, A, ncol, s, 0ull, apply_bytes));
      CKL();
      CK(cudaMemcpyAsync(ctx->h_flag, &e.st->any_active, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (!*ctx->h_flag) break;
    }
    return launch_tail_shard(ctx, bl, e, A, ncol, cfg->logdet_mode, s, apply_bytes);
  }
  while (done < limit) {
    for (int q = 0; q < CH && done < limit; ++q, ++done) {
      if (A.lowrank) PROF(ctx, PC_OTHER, 0.0, s, launch_lowrank(A.t1, A.ncp, s));
      PROF(ctx, apply_cls, apply_bytes, s, launch_apply(A.a1, A.ncp, s));
      if (!A.mbcg) {
        if (A.lowrank) PROF(ctx, PC_OTHER, 0.0, s, launch_lowrank(A.t2, A.ncp, s));
        PROF(ctx, apply_cls, apply_bytes, s, launch_apply(A.a2, A.ncp, s));
      }
      PROF(ctx, PC_UPDATE, 0.0, s, launch_update(A.ua, A.ncp, s));
    }
    CKL();
    CK(cudaMemcpyAsync(ctx->h_flag, &e.st->any_active, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!*ctx->h_flag) break;
  }
  if (A.mbcg) {
    launch_tail_final(bl, e, A, ncol, cfg->logdet_mode, s);
  } else {
    launch_spart(Ld, B.u, e.X, ncol, e.SX, s);
    if (A.lowrank) PROF(ctx, PC_OTHER, 0.0, s, launch_lowrank(A.t3, A.ncp, s));
    PROF(ctx, apply_cls, apply_bytes, s, launch_apply(A.a3, A.ncp, s));
    if (A.lowrank) PROF(ctx, PC_OTHER, 0.0, s, launch_lowrank(A.t4, A.ncp, s));
    PROF(ctx, apply_cls, apply_bytes, s, launch_apply(A.a4, A.ncp, s));
    launch_final(e.st, e.prm, e.ah, e.bh, HIST, e.slqw, B.scal + 0, static_cast<double>(L.n),
                 ncol, cfg->logdet_mode, e.out, s);
  }
  CKL();
  return NUGPR_OK;
}

static nugpr_status get_graph(nugpr_ctx* ctx, nugpr_blocks* bl, int slot, int ncol, int logdet_mode,
                              cudaGraphExec_t* out) {
  const std::string key = graph_key(bl, slot, ncol, logdet_mode);
  auto it = ctx->graphs.find(key);
  if (it != ctx->graphs.end()) { *out = it->second; return NUGPR_OK; }
  EvalDev& e = bl->E[slot];
  IterArgs A;
  RET(make_iter_args(bl, e, ncol, A, logdet_mode == NUGPR_LOGDET_MBCG));
  // every kernel of the graph opts into its shared memory before capture
  cudaStream_t cs = ctx->capture_stream;
  cudaGraph_t g = nullptr;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wnode;
  CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  A.ua.cond = h;
  CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  nugpr_status cst = NUGPR_OK;
  if (bl->shard) {
    A.ua.cond = 0;                                 // (FIN_UPDATE after the exchange sets the condition)
    cst = launch_iteration_shard(ctx, bl, e, A, ncol, cs, h);
  } else {
    launch_iteration(A, cs);
  }
  cudaGraph_t body_out = nullptr;
  cudaError_t ce = cudaStreamEndCapture(cs, &body_out);
  if (cst != NUGPR_OK) { cudaGraphDestroy(g); return cst; }
  if (ce != cudaSuccess) { cudaGraphDestroy(g); return fail(NUGPR_ERR_CUDA, "graph body capture: %s", cudaGetErrorString(ce)); }
  CK(cudaStreamBeginCaptureToGraph(cs, g, &wnode, nullptr, 1, cudaStreamCaptureModeRelaxed));
  if (bl->shard) cst = launch_tail_shard(ctx, bl, e, A, ncol, logdet_mode, cs);
  else launch_tail_final(bl, e, A, ncol, logdet_mode, cs);
  cudaGraph_t g_out = nullptr;
  ce = cudaStreamEndCapture(cs, &g_out);
  if (cst != NUGPR_OK) { cudaGraphDestroy(g); return cst; }
  if (ce != cudaSuccess) { cudaGraphDestroy(g); return fail(NUGPR_ERR_CUDA, "graph tail capture: %s", cudaGetErrorString(ce)); }
  cudaGraphExec_t ex = nullptr;
  ce = cudaGraphInstantiate(&ex, g, 0);
  if (ce != cudaSuccess) { cudaGraphDestroy(g); return fail(NUGPR_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ce)); }
  ctx->graphs[key] = ex;
  ctx->graph_defs.push_back(g);
  *out = ex;
  return NUGPR_OK;
}

static nugpr_status check_cfg(const nugpr_solve_cfg* cfg) {
  if (!cfg) return fail(NUGPR_ERR_INVALID_ARG, "cfg is NULL");
  if (cfg->num_probes < 1 || cfg->num_probes > NUGPR_MAX_PROBES)
    return fail(NUGPR_ERR_INVALID_ARG, "num_probes must be in [1, %d]", NUGPR_MAX_PROBES);
  if (cfg->cg_max_iter < 1 || cfg->cg_max_iter >= HIST)
    return fail(NUGPR_ERR_INVALID_ARG, "cg_max_iter must be in [1, %d)", HIST);
  if (!(cfg->cg_tol >= 0.0)) return fail(NUGPR_ERR_INVALID_ARG, "cg_tol must be >= 0");
  if (cfg->logdet_mode < 0 || cfg->logdet_mode > 2) return fail(NUGPR_ERR_INVALID_ARG, "bad logdet_mode");
  return NUGPR_OK;
}

static nugpr_status stage_y(nugpr_blocks* bl, const double* y, cudaStream_t s, const double** y_dev) {
  if (is_device_ptr(y)) { *y_dev = y; return NUGPR_OK; }
  CK(cudaMemcpyAsync(bl->B.ystage, y, sizeof(double) * bl->n_glob, cudaMemcpyHostToDevice, s));
  *y_dev = bl->B.ystage;
  return NUGPR_OK;
}

// Kernel launches a finished graph-mode evaluation made (host counter for gpu_launches).
static void account_graph_launches(const nugpr_blocks* bl, const nugpr_mll_out& o, int logdet_mode) {
  int k = o.iters_y;
  for (int j = 0; j < 16; ++j) k = std::max(k, o.iters_q[j]);
  const bool mb = logdet_mode == NUGPR_LOGDET_MBCG;
  // per iteration: apply (+ apply) + update, + a lowrank before each apply in the big-block layout;
  // tail: spart + 2 applies (+ 2 lowrank) + final, or quad_part + final (mBCG)
  const bool lr = bl->L.big;
  const long long per_it = (mb ? 2 : 3) + (lr ? (mb ? 1 : 2) : 0);
  note_launch(per_it * std::max(1, k) + (mb ? 2 : (lr ? 6 : 4)));
}

static nugpr_status finish_record(nugpr_blocks* bl, const nugpr_solve_cfg* cfg, const nugpr_mll_out& o,
                                  bool graph) {
  if (graph) account_graph_launches(bl, o, cfg->logdet_mode);
  bl->last_m = cfg->num_probes;
  bl->last_seed = cfg->probe_seed;
  if (!o.lanczos_converged)
    return fail(NUGPR_ERR_INTERNAL, "lambda_0 Lanczos did not converge in %d iterations", o.lanczos_iters);
  if (!(o.lambda0 > 0.0) || o.lambda0_degenerate)
    return fail(NUGPR_ERR_DEGENERATE_REPS, "lambda_0(theta) = %g is not certifiably > 0", o.lambda0);
  if (o.breakdown)
    return fail(NUGPR_ERR_BREAKDOWN, "CG breakdown: non-finite r^T r or non-positive / non-finite p^T q");
  if (!o.converged) return fail(NUGPR_ERR_CG_NOT_CONVERGED, "CG reached cg_max_iter = %d", cfg->cg_max_iter);
  return NUGPR_OK;
}

// One evaluation on the context stream with slot 0, record read back.
static nugpr_status run_eval(nugpr_ctx* ctx, nugpr_blocks* bl, const double* y_dev, nugpr_theta th,
                             const nugpr_solve_cfg* cfg, nugpr_mll_out* out) {
  cudaStream_t s = ctx->stream;
  cudaGetLastError();
  int mode = 0;
  RET(enqueue_eval(ctx, bl, 0, y_dev, th, cfg, s, &mode, &ctx->h_prm[0]));
  CK(cudaMemcpyAsync(&ctx->h_out[0], bl->E[0].out, sizeof(nugpr_mll_out), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  prof_harvest(ctx);
  *out = ctx->h_out[0];
  return finish_record(bl, cfg, *out, !ctx->prof && ctx->use_graphs);
}

extern "C" nugpr_status nugpr_mll(nugpr_ctx* ctx, nugpr_blocks* bl, const double* y_sorted, nugpr_theta theta,
                                  const nugpr_solve_cfg* cfg, nugpr_mll_out* out) {
  if (!ctx || !bl || !y_sorted || !out) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  if (!theta_ok(theta)) return fail(NUGPR_ERR_INVALID_ARG, "theta must be positive and finite");
  RET(check_cfg(cfg));
  CK(cudaSetDevice(ctx->device));
  const double* y_dev = nullptr;
  RET(stage_y(bl, y_sorted, ctx->stream, &y_dev));
  bl->cy_ready = false;
  return run_eval(ctx, bl, y_dev, theta, cfg, out);
}

// ------------------------------------------------------------------------------------------
// Numerical gradient (row A8).
extern "C" nugpr_status nugpr_shard_plan(int32_t world, const double* costs, int32_t n, int32_t* owner) {
  if (world < 1 || n < 0 || (n > 0 && (!costs || !owner))) return fail(NUGPR_ERR_INVALID_ARG, "bad shard plan args");
  std::vector<int> idx(n);
  for (int k = 0; k < n; ++k) idx[k] = k;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return costs[a] > costs[b]; });
  std::vector<double> load(world, 0.0);
  for (int k : idx) {
    int best = 0;
    for (int r = 1; r < world; ++r) if (load[r] < load[best]) best = r;
    owner[k] = best;
    load[best] += costs[k];
  }
  return NUGPR_OK;
}

struct EvalRecord {
  nugpr_mll_out o;
  int32_t status;
  int32_t valid;
};

// Status of a set of evaluation records: the first hard failure (in evaluation order) wins over
// CG non-convergence ("flag any instances"), which wins over OK.
static nugpr_status worst_status(const EvalRecord* recs, int n, int* which) {
  nugpr_status w = NUGPR_OK;
  *which = -1;
  for (int k = 0; k < n; ++k) {
    const nugpr_status st = static_cast<nugpr_status>(recs[k].status);
    if (st == NUGPR_OK) continue;
    if (st != NUGPR_ERR_CG_NOT_CONVERGED) { *which = k; return st; }
    if (w == NUGPR_OK) { w = st; *which = k; }
  }
  return w;
}

// PAR-1 exchange of the CENTRAL gradient: every rank holds the records of the
// evaluations it owns (owner[k] == rank); one allgather of the 7-record arrays, then each record
// is taken from its owner's copy, and every rank forms the same L0 and g_i = (L+ - L-)/(2 h_i)
// (Eq. 11 read as a central difference, reading X2).
static nugpr_status central_exchange(nugpr_ctx* ctx, const int32_t* owner, const EvalRecord* mine,
                                     const double* h, double* L0, double* grad, nugpr_mll_out* evals,
                                     nugpr_status* worst, int world) {
  EvalRecord all[NUGPR_NUM_EVALS];
  if (world > 1 && ctx->nccl) {
    // in-library NCCL: the records through the context's device scratch (one host sync)
    const size_t nb = sizeof(EvalRecord) * NUGPR_NUM_EVALS;
    if (nb * static_cast<size_t>(world) > 65536) return fail(NUGPR_ERR_INTERNAL, "record exchange scratch too small");
    char* d = static_cast<char*>(ctx->nccl_scratch);
    std::vector<EvalRecord> recv(static_cast<size_t>(world) * NUGPR_NUM_EVALS);
    CK(cudaMemcpyAsync(d, mine, nb, cudaMemcpyHostToDevice, ctx->stream));
    const NcclRT& rt = nccl_rt();
    const ncclResult_t r = rt.AllGather(d, d + nb, nb, ncclUint8, ctx->nccl, ctx->stream);
    if (r != ncclSuccess) return fail(NUGPR_ERR_COMM, "ncclAllGather: %s", rt.GetErrorString(r));
    CK(cudaMemcpyAsync(recv.data(), d + nb, nb * world, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < NUGPR_NUM_EVALS; ++k) all[k] = recv[static_cast<size_t>(owner[k]) * NUGPR_NUM_EVALS + k];
  } else if (world > 1) {
    if (!ctx->ag) return fail(NUGPR_ERR_COMM, "world > 1 but no allgather callback set");
    std::vector<EvalRecord> recv(static_cast<size_t>(ctx->world) * NUGPR_NUM_EVALS);
    if (ctx->ag(mine, sizeof(EvalRecord) * NUGPR_NUM_EVALS, recv.data(), ctx->ag_user) != 0)
      return fail(NUGPR_ERR_COMM, "allgather failed");
    for (int k = 0; k < NUGPR_NUM_EVALS; ++k) all[k] = recv[static_cast<size_t>(owner[k]) * NUGPR_NUM_EVALS + k];
  } else {
    memcpy(all, mine, sizeof(all));
  }
  for (int k = 0; k < NUGPR_NUM_EVALS; ++k) {
    if (!all[k].valid) return fail(NUGPR_ERR_COMM, "evaluation %d missing after exchange", k);
    if (evals) evals[k] = all[k].o;
  }
  int which = -1;
  *worst = worst_status(all, NUGPR_NUM_EVALS, &which);
  if (*worst != NUGPR_OK)
    fail(*worst, "central-difference evaluation %d (0 = theta, 1+2i / 2+2i = theta +- h_i e_i) ended with status %d "
                 "(rank %d owned it)", which, static_cast<int>(*worst), owner[which]);
  *L0 = all[0].o.L;
  for (int i = 0; i < 3; ++i) grad[i] = (all[1 + 2 * i].o.L - all[2 + 2 * i].o.L) / (2.0 * h[i]);
  return NUGPR_OK;
}

// Host-only entry to the same exchange (tests of the sharded path without a GPU): this rank
// passes L values for the evaluations nugpr_shard_plan gives it (others ignored).
extern "C" nugpr_status nugpr_numgrad_exchange(nugpr_ctx* ctx, nugpr_theta theta, const double step[3],
                                               const double L_mine[7], const int32_t* status_mine, double* L0,
                                               double grad[3]) {
  if (!ctx || !step || !L_mine || !L0 || !grad) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  const double th[3] = {theta.lengthscale, theta.noise, theta.outputscale};
  double h[3];
  for (int i = 0; i < 3; ++i) h[i] = step[i] * th[i];
  const double cost[NUGPR_NUM_EVALS] = {1.0, 3.0, 3.0, 2.0, 2.0, 2.0, 2.0};
  int32_t owner[NUGPR_NUM_EVALS];
  RET(nugpr_shard_plan(ctx->world, cost, NUGPR_NUM_EVALS, owner));
  EvalRecord mine[NUGPR_NUM_EVALS];
  memset(mine, 0, sizeof(mine));
  for (int k = 0; k < NUGPR_NUM_EVALS; ++k)
    if (owner[k] == ctx->rank) {
      mine[k].o.L = L_mine[k];
      mine[k].valid = 1;
      mine[k].status = status_mine ? status_mine[k] : NUGPR_OK;
    }
  nugpr_status worst = NUGPR_OK;
  RET(central_exchange(ctx, owner, mine, h, L0, grad, nullptr, &worst, ctx->world));
  return worst;
}

// Evaluate the points `ks` (indices into pts) concurrently: evaluation j runs on slot j % slots,
// each slot on its own stream forked from the context stream; one host sync at the end.
static nugpr_status run_evals_concurrent(nugpr_ctx* ctx, nugpr_blocks* bl, const double* y_dev,
                                         const std::vector<int>& ks, const nugpr_theta* pts,
                                         const nugpr_solve_cfg* cfg, EvalRecord* recs) {
  cudaStream_t s0 = ctx->stream;
  const int slots = static_cast<int>(bl->E.size());
  const bool graph = !ctx->prof && ctx->use_graphs;
  // Every evaluation gets a record and a status, whatever happens to the others: nugpr_numgrad
  // always reaches the PAR-1 exchange afterwards, so no rank is left waiting in it (a rank that
  // returned early would deadlock the others' allgather).
  auto mark_rest = [&](size_t from, nugpr_status st) {
    for (size_t q = from; q < ks.size(); ++q) { recs[ks[q]].status = st; recs[ks[q]].valid = 1; }
  };
  if (slots <= 1 || ctx->prof || ks.size() <= 1 || bl->shard) {
    for (int k : ks) {
      nugpr_status st = run_eval(ctx, bl, y_dev, pts[k], cfg, &recs[k].o);
      recs[k].status = st;
      recs[k].valid = 1;
    }
    return NUGPR_OK;
  }
  {
    const nugpr_status ss_ = ensure_slot_streams(ctx, slots);
    if (ss_ != NUGPR_OK) { mark_rest(0, ss_); return NUGPR_OK; }
  }
  const int nk = static_cast<int>(ks.size());
  if (cfg->block_storage == NUGPR_BLOCKS_F32 && !bl->h32_ready && !bl->L.big) {
    if (bl->h_pending) CK(cudaStreamWaitEvent(s0, ctx->ev_h1, 0));
    launch_d2f(bl->B.H, bl->B.H32, bl->L.pk_total, s0);    // before the fork: every stream reads it
    CKL();
    bl->h32_ready = true;
  }
  CK(cudaEventRecord(ctx->ev_fork, s0));
  int modes[16] = {0};
  int q = 0;                                         // stream index of the next job
  // an enqueue failure ends the launching (that job and the ones not yet launched carry its status);
  // the jobs already in flight are still joined and read back
  nugpr_status enq = NUGPR_OK;
  int failed_at = nk;
  auto note_enq = [&](nugpr_status st, int j) { if (st != NUGPR_OK && enq == NUGPR_OK) { enq = st; failed_at = j; } };
  std::vector<char> launched(nk, 0);
  for (int j = 0; j < nk && enq == NUGPR_OK; ++j) {
    const int slot = j % slots;
    cudaStream_t ss = ctx->slot_stream[q % slots];
    if (q < slots) note_enq(cudaStreamWaitEvent(ss, ctx->ev_fork, 0) == cudaSuccess ? NUGPR_OK
                            : fail(NUGPR_ERR_CUDA, "stream fork failed"), j);
    ++q;
    if (enq != NUGPR_OK) break;
    note_enq(enqueue_eval(ctx, bl, slot, y_dev, pts[ks[j]], cfg, ss, &modes[j], &ctx->h_prm[j]), j);
    if (enq != NUGPR_OK) break;
    note_enq(cudaMemcpyAsync(&ctx->h_out[j], bl->E[slot].out, sizeof(nugpr_mll_out), cudaMemcpyDeviceToHost, ss)
                     == cudaSuccess ? NUGPR_OK : fail(NUGPR_ERR_CUDA, "record read-back failed"), j);
    if (enq == NUGPR_OK) launched[j] = 1;
  }
  for (int slot = 0; slot < std::min(slots, q); ++slot) {
    cudaEventRecord(ctx->ev_join[slot], ctx->slot_stream[slot]);
    cudaStreamWaitEvent(s0, ctx->ev_join[slot], 0);
  }
  const cudaError_t se = cudaStreamSynchronize(s0);
  if (se != cudaSuccess) {
    mark_rest(0, fail(NUGPR_ERR_CUDA, "evaluation streams: %s", cudaGetErrorString(se)));
    return NUGPR_OK;
  }
  for (int j = 0; j < nk; ++j) {
    EvalRecord& r = recs[ks[j]];
    r.valid = 1;
    if (launched[j]) {
      r.o = ctx->h_out[j];
      r.status = finish_record(bl, cfg, r.o, graph);
    } else {
      memset(&r.o, 0, sizeof(r.o));
      r.o.L = NAN;
      r.status = (j >= failed_at) ? enq : NUGPR_ERR_INTERNAL;
    }
  }
  return NUGPR_OK;
}


extern "C" nugpr_status nugpr_numgrad(nugpr_ctx* ctx, nugpr_blocks* bl, const double* y_sorted, nugpr_theta theta,
                                      const nugpr_grad_cfg* gcfg, const nugpr_solve_cfg* scfg, double* L0,
                                      double grad[3], nugpr_mll_out* evals, int32_t* n_evals) {
  if (!ctx || !bl || !y_sorted || !gcfg || !L0 || !grad) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  if (!theta_ok(theta)) return fail(NUGPR_ERR_INVALID_ARG, "theta must be positive and finite");
  RET(check_cfg(scfg));
  CK(cudaSetDevice(ctx->device));
  cudaGetLastError();
  const double th[3] = {theta.lengthscale, theta.noise, theta.outputscale};
  const double* y_dev = nullptr;
  RET(stage_y(bl, y_sorted, ctx->stream, &y_dev));
  auto mk = [](const double* p) { nugpr_theta t{p[0], p[1], p[2]}; return t; };
  int ne = 0;
  // every evaluation of this call shares y and R: c = R^{-T} y is computed once and reused
  struct CyGuard { nugpr_blocks* b; ~CyGuard() { b->cy_ready = false; } } cyg{bl};
  launch_cy(bl->Ld, bl->B.Linv, y_dev + bl->pos0, bl->L.ld_max, bl->B.cy, ctx->stream);
  CKL();
  bl->cy_ready = true;
  if (gcfg->mode == NUGPR_GRAD_CENTRAL) {
    double pts[NUGPR_NUM_EVALS][3];
    double h[3];
    for (int i = 0; i < 3; ++i) h[i] = gcfg->step[i] * th[i];
    for (int k = 0; k < NUGPR_NUM_EVALS; ++k) for (int i = 0; i < 3; ++i) pts[k][i] = th[i];
    for (int i = 0; i < 3; ++i) {
      pts[1 + 2 * i][i] = th[i] + h[i];
      pts[2 + 2 * i][i] = th[i] - h[i];
      if (!(pts[2 + 2 * i][i] > 0.0)) return fail(NUGPR_ERR_INVALID_ARG, "step too large for parameter %d", i);
    }
    nugpr_theta tp[NUGPR_NUM_EVALS];
    for (int k = 0; k < NUGPR_NUM_EVALS; ++k) tp[k] = mk(pts[k]);
    // perturbation sharding (PAR-1): LPT over a cost model (baseline: no block reads; lambda:
    // G precompute + Lanczos)
    const double cost[NUGPR_NUM_EVALS] = {1.0, 3.0, 3.0, 2.0, 2.0, 2.0, 2.0};
    int32_t owner[NUGPR_NUM_EVALS];
    // (PAR-2 sharded blocks: every rank takes part in every evaluation, so no perturbation split)
    const int pw = bl->shard ? 1 : ctx->world, pr = bl->shard ? 0 : ctx->rank;
    RET(nugpr_shard_plan(pw, cost, NUGPR_NUM_EVALS, owner));
    EvalRecord mine[NUGPR_NUM_EVALS];
    memset(mine, 0, sizeof(mine));
    std::vector<int> ks;                       // this rank's evaluations, most expensive first
    for (int k : {1, 2, 3, 4, 5, 6, 0}) if (owner[k] == pr) ks.push_back(k);
    RET(run_evals_concurrent(ctx, bl, y_dev, ks, tp, scfg, mine));   // statuses live in the records
    // every rank exchanges, failed evaluations included (their status travels with the record)
    nugpr_status worst = NUGPR_OK;
    RET(central_exchange(ctx, owner, mine, h, L0, grad, evals, &worst, pw));
    ne = NUGPR_NUM_EVALS;
    if (n_evals) *n_evals = ne;
    if (worst != NUGPR_OK) return worst;     // central_exchange set the message
    return NUGPR_OK;
  } else if (gcfg->mode == NUGPR_GRAD_FORWARD_HALVING) {
    if (gcfg->max_halvings < 0 || gcfg->max_halvings > 20) return fail(NUGPR_ERR_INVALID_ARG, "max_halvings must be in [0, 20]");
    // Alg. 1 lines 265-278 (readings P12-P14)
    nugpr_mll_out o;
    nugpr_status st = run_eval(ctx, bl, y_dev, theta, scfg, &o);
    if (st != NUGPR_OK) return st;
    if (evals) evals[ne] = o;
    ++ne;
    *L0 = o.L;
    for (int i = 0; i < 3; ++i) {
      double delta = gcfg->step[i] * th[i];
      double gprev = INFINITY, g = 0.0;
      int nh = 0;
      while (true) {
        double p[3] = {th[0], th[1], th[2]};
        p[i] += delta;
        nugpr_mll_out o1;
        st = run_eval(ctx, bl, y_dev, mk(p), scfg, &o1);
        if (st != NUGPR_OK) return st;
        if (evals) evals[ne] = o1;
        ++ne;
        g = (o1.L - o.L) / delta;
        const double scale = gcfg->threshold_relative ? std::max(1.0, std::fabs(g)) : 1.0;
        if (std::fabs(g - gprev) < gcfg->threshold * scale || nh >= gcfg->max_halvings) break;
        gprev = g;
        delta *= 0.5;
        ++nh;
      }
      grad[i] = g;
    }
    if (n_evals) *n_evals = ne;
    return NUGPR_OK;
  }
  return fail(NUGPR_ERR_INVALID_ARG, "bad gradient mode");
}

// ------------------------------------------------------------------------------------------
// NEXT-1: posterior mean / variance (Eq. 4-5) with the exact structured K''^{-1} (predict_kernels.cu).
// The capacitance matrix of Eq. (28)'s Woodbury form (reading P22): with c = R^{-T} y in B.cy,
// zeta_i = u_i^T c_i / sqrt(d_i) -> e.Tbuf[0:n_c], sqrt(d_i) -> e.Tbuf[n_c:2n_c];
// C = I + D^{1/2} M D^{1/2} (one ldc x ldc block in e.V), factorised in place to Linv_C with
// log|C| -> e.scal[0]; lz = Linv_C zeta -> e.Tbuf[2n_c:3n_c].  Small (fused) or blocked big-block
// factorisation by size.  Synchronises the stream (reads the SPD status).
static nugpr_status factor_capacitance(nugpr_blocks* bl, EvalDev& e, const double* c, int ldc, cudaStream_t s) {
  const HostLayout& L = bl->L;
  BlocksDev& B = bl->B;
  const int n_c = L.n_c;
  const bool big = ldc > LD_SMALL_MAX;
  double* Cm = B.cap;                     // its own workspace region (any n_c)
  double* zeta = e.Tbuf, *sd = e.Tbuf + n_c, *lz = e.Tbuf + 2 * n_c;
  launch_pred_setup(bl->Ld, c, B.u, B.M, ldc, zeta, sd, Cm, s);
  int64_t hm[16] = {0, n_c, 0, ldc, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};   // off[2], poff[2], boff[1]
  int32_t* ldp = reinterpret_cast<int32_t*>(B.pmeta + 8);                     // ld[1]
  int32_t ldh = ldc;
  std::memcpy(&hm[8], &ldh, sizeof(int32_t));
  CK(cudaMemcpyAsync(B.pmeta, hm, sizeof(hm), cudaMemcpyHostToDevice, s));
  LayoutDev Lc = bl->Ld;
  Lc.off = B.pmeta; Lc.poff = B.pmeta + 2; Lc.boff = B.pmeta + 4; Lc.ld = ldp; Lc.n_c = 1;
  if (big) launch_big_chol_trtri(Cm, Lc, nullptr, 0, ldc, e.linfo, e.scal, e.U, B.capscr, s);
  else launch_chol_trtri(Cm, Lc, nullptr, 0, ldc, e.linfo, e.scal, e.U, s);
  CKL();
  int32_t cst = 0;
  CK(cudaMemcpyAsync(&cst, e.linfo, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  launch_pred_lz(Cm, ldc, n_c, zeta, lz, s);
  CKL();
  CK(cudaStreamSynchronize(s));
  if (cst) return fail(NUGPR_ERR_NOT_SPD, "I + M~ is not SPD (degenerate low-rank term)");
  return NUGPR_OK;
}

extern "C" nugpr_status nugpr_predict(nugpr_ctx* ctx, nugpr_blocks* bl, const double* y_sorted, const double* X_test,
                                      int64_t n_test, int32_t add_noise, double* mean, double* var) {
  if (!ctx || !bl || !y_sorted || !X_test || !mean) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  if (n_test < 0) return fail(NUGPR_ERR_INVALID_ARG, "n_test < 0");
  if (bl->shard) return fail(NUGPR_ERR_UNSUPPORTED, "predict needs replicated (unsharded) blocks");
  if (n_test == 0) return NUGPR_OK;
  const HostLayout& L = bl->L;
  CK(cudaSetDevice(ctx->device));
  cudaGetLastError();
  cudaStream_t s = ctx->stream;
  const LayoutDev& Ld = bl->Ld;
  BlocksDev& B = bl->B;
  EvalDev& e = bl->E[0];
  const int n_c = L.n_c, d = L.d;
  const int ldc = (n_c + PAD - 1) / PAD * PAD;
  const nugpr_theta th = bl->theta0;
  // chunk of test points bounded by the slot buffers it uses
  int64_t nt = 256;
  nt = std::min<int64_t>(nt, L.blk_total / std::max<int64_t>(1, L.n_pad));
  nt = std::min<int64_t>(nt, (static_cast<int64_t>(MAXC) * L.n_pad) / (3 * std::max(n_c, ldc)));
  nt = std::min<int64_t>(nt, (static_cast<int64_t>(MAXC) * L.n_pad) / std::max(1, d));
  if (nt < 1) return fail(NUGPR_ERR_WORKSPACE, "workspace too small for predict");
  double* Ks = e.G;                       // n_pad x nt (per-cluster column-major)
  double* W = e.T;                        // same layout
  double* wc = e.RHS;                     // [n_c][nt] x 3
  double* ww = wc + static_cast<int64_t>(n_c) * nt;
  double* p = ww + static_cast<int64_t>(n_c) * nt;
  double* pc = e.R;                       // ldc x nt
  double* lp = e.X;                       // ldc x nt
  double* Cm = B.cap;                     // ldc x ldc (C, then Linv_C): factor_capacitance
  double* zeta = e.Tbuf, *lz = e.Tbuf + 2 * n_c;
  double* xt = e.Q;                       // nt x d staged test inputs
  double* ostage = e.dots;                // 2 * nt outputs when the user's buffers are host memory
  // c = R^{-T} y
  const double* y_dev = nullptr;
  RET(stage_y(bl, y_sorted, s, &y_dev));
  launch_cy(Ld, B.Linv, y_dev, L.ld_max, B.cy, s);
  RET(factor_capacitance(bl, e, B.cy, ldc, s));
  int32_t* ldp = reinterpret_cast<int32_t*>(B.pmeta + 8);                     // ld[1] of the one-block layout
  int64_t* zero64 = B.pmeta + 10;                                             // loff = goff = 0
  const bool xdev = is_device_ptr(X_test), mdev = is_device_ptr(mean), vdev = var ? is_device_ptr(var) : true;
  const double noise_add = add_noise ? th.noise : 0.0;
  for (int64_t j0 = 0; j0 < n_test; j0 += nt) {
    const int m = static_cast<int>(std::min<int64_t>(nt, n_test - j0));
    const double* xtp = X_test + j0 * d;
    if (!xdev) {
      CK(cudaMemcpyAsync(xt, xtp, sizeof(double) * m * d, cudaMemcpyHostToDevice, s));
      xtp = xt;
    }
    launch_pred_ks(B.X, xtp, d, Ld, m, L.ld_max, bl->kind, th.lengthscale, th.outputscale, Ks, s);
    launch_pred_trmm(B.Linv, Ks, W, B.ld, B.boff, B.poff, n_c, m, L.ld_max, s);
    launch_pred_reduce(Ld, W, B.cy, B.u, m, wc, ww, p, s);
    launch_pred_pcol(p, n_c, m, ldc, pc, s);
    launch_pred_trmm(Cm, pc, lp, ldp, zero64, zero64, 1, m, ldc, s);
    // device outputs are written in place at offset j0; host outputs go through the staging area
    // (mean at ostage[0..m), var at ostage[nt..nt+m)) and are copied out below — independently per output
    double* mo = mdev ? mean : ostage;
    double* vo = var ? (vdev ? var : ostage + nt) : nullptr;
    launch_pred_final(n_c, m, ldc, wc, ww, pc, lp, zeta, lz, th.outputscale, noise_add, mo, vo,
                      mdev ? j0 : 0, vdev ? j0 : 0, s);
    CKL();
    if (!mdev) CK(cudaMemcpyAsync(mean + j0, ostage, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    if (var && !vdev) CK(cudaMemcpyAsync(var + j0, ostage + nt, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    if (!mdev || (var && !vdev) || !xdev) CK(cudaStreamSynchronize(s));
  }
  CK(cudaStreamSynchronize(s));
  return NUGPR_OK;
}


// ------------------------------------------------------------------------------------------
// NEXT-2: the exact structured MLL at the blocks' theta_0 (Eq. (28)-(29)):
// determinant lemma + Woodbury on the rank-n_c term, no probes / Pade / CG.
extern "C" nugpr_status nugpr_mll_exact(nugpr_ctx* ctx, nugpr_blocks* bl, const double* y_sorted, double out[4]) {
  if (!ctx || !bl || !y_sorted || !out) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  if (bl->shard) return fail(NUGPR_ERR_UNSUPPORTED, "mll_exact needs replicated (unsharded) blocks");
  CK(cudaSetDevice(ctx->device));
  cudaGetLastError();
  cudaStream_t s = ctx->stream;
  const HostLayout& L = bl->L;
  BlocksDev& B = bl->B;
  EvalDev& e = bl->E[0];
  const int ldc = (L.n_c + PAD - 1) / PAD * PAD;
  const double* y_dev = nullptr;
  RET(stage_y(bl, y_sorted, s, &y_dev));
  launch_cy(bl->Ld, B.Linv, y_dev, L.ld_max, B.cy, s);
  bl->cy_ready = false;                          // B.cy now holds this y's c (numgrad recomputes its own)
  CKL();
  RET(factor_capacitance(bl, e, B.cy, ldc, s));
  double* ccblk = e.Tbuf + 3 * L.n_c;
  double* dout = e.scal + 4;
  launch_exact_final(bl->Ld, B.cy, e.Tbuf, e.Tbuf + 2 * L.n_c, B.scal, e.scal, ccblk, L.n, dout, s);
  CKL();
  CK(cudaMemcpyAsync(ctx->h_out, dout, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::memcpy(out, ctx->h_out, 4 * sizeof(double));
  return NUGPR_OK;
}
// ------------------------------------------------------------------------------------------
extern "C" nugpr_status nugpr_adam_step(double state[10], const double grad[3], double lr) {
  if (!state || !grad) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  for (int i = 0; i < 3; ++i)
    if (!std::isfinite(grad[i]))    // (a NaN would otherwise pass the clamp below as 1e-8 and poison m, v)
      return fail(NUGPR_ERR_INVALID_ARG, "non-finite gradient component %d (%g): Adam step refused", i, grad[i]);
  for (int i = 0; i < 9; ++i)
    if (!std::isfinite(state[i])) return fail(NUGPR_ERR_INVALID_ARG, "non-finite Adam state entry %d", i);
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  double t = state[9] + 1.0;
  for (int i = 0; i < 3; ++i) {
    double m = b1 * state[3 + i] + (1.0 - b1) * grad[i];
    double v = b2 * state[6 + i] + (1.0 - b2) * grad[i] * grad[i];
    double mh = m / (1.0 - std::pow(b1, t));
    double vh = v / (1.0 - std::pow(b2, t));
    double th = state[i] - lr * mh / (std::sqrt(vh) + eps);
    state[i] = th > 1e-8 ? th : 1e-8;
    state[3 + i] = m;
    state[6 + i] = v;
  }
  state[9] = t;
  return NUGPR_OK;
}

extern "C" nugpr_status nugpr_train(nugpr_ctx* ctx, const double* X_sorted, const int64_t* offsets, int32_t n_c,
                                    int32_t d, const double* reps, const double* y_sorted, int32_t kernel,
                                    int32_t epochs, double lr, const nugpr_grad_cfg* gcfg,
                                    const nugpr_solve_cfg* scfg, double adam_state[10], double* records,
                                    void* workspace, size_t ws_bytes) {
  if (!ctx || !adam_state || !gcfg || !scfg) return fail(NUGPR_ERR_INVALID_ARG, "NULL argument");
  if (epochs < 0) return fail(NUGPR_ERR_INVALID_ARG, "epochs < 0");
  for (int ep = 0; ep < epochs; ++ep) {
    nugpr_theta th{adam_state[0], adam_state[1], adam_state[2]};
    nugpr_blocks* bl = nullptr;
    int32_t fb = -1;
    double jit = 0.0;
    RET(build_impl(ctx, X_sorted, offsets, n_c, d, reps, kernel, th, workspace, ws_bytes, &bl, &fb, &jit, ep > 0,
                   true));
    double L0 = 0.0, g[3] = {0, 0, 0};
    nugpr_mll_out ev[1 + 3 * 21];
    int32_t ne = 0;
    nugpr_status st = nugpr_numgrad(ctx, bl, y_sorted, th, gcfg, scfg, &L0, g, ev, &ne);
    if (bl->h_pending) cudaStreamWaitEvent(ctx->stream, ctx->ev_h1, 0);   // H done before the next build
    nugpr_blocks_destroy(bl);
    if (st != NUGPR_OK) return st;
    if (!std::isfinite(L0)) return fail(NUGPR_ERR_BREAKDOWN, "epoch %d: non-finite loss L0 = %g", ep, L0);
    if (records) {
      double* r = records + static_cast<size_t>(ep) * NUGPR_TRAIN_RECORD;
      int ky = 0, kq = 0;
      for (int k = 0; k < ne; ++k) { ky = std::max(ky, ev[k].iters_y); kq = std::max(kq, ev[k].iters_q_max); }
      r[0] = L0; r[1] = g[0]; r[2] = g[1]; r[3] = g[2];
      r[4] = th.lengthscale; r[5] = th.noise; r[6] = th.outputscale;
      r[7] = ky; r[8] = kq; r[9] = jit; r[10] = ne; r[11] = 0.0;
    }
    RET(nugpr_adam_step(adam_state, g, lr));
  }
  return NUGPR_OK;
}

extern "C" nugpr_status nugpr_tridiag_eig(int32_t k, const double* diag, const double* off, double* evals,
                                          double* first) {
  if (k < 1 || !diag || !evals || !first || (k > 1 && !off)) return fail(NUGPR_ERR_INVALID_ARG, "bad args");
  std::vector<double> e(k, 0.0);
  for (int i = 0; i + 1 < k; ++i) e[i] = off[i];
  for (int i = 0; i < k; ++i) evals[i] = diag[i];
  if (tql_first(k, evals, e.data(), first) != 0) return fail(NUGPR_ERR_INTERNAL, "QL did not converge");
  return NUGPR_OK;
}
