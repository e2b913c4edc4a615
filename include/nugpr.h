/*
 * nugpr.h — C-ABI of the B200-native nuGPR training hot path (arXiv 2510.12128).
 *
 * The library (libnugpr.so, hand-written sm_100a CUDA) evaluates the negative marginal
 * log-likelihood of a GP on clustered inputs (Eq. 3, lines 59-62) with the
 * paper's structured covariance K'' (Eq. 28), the block-Cholesky
 * preconditioner R (Eq. 12-13), batched multi-RHS PCG (PAPER.md:107-108,
 * 124), the Hutchinson / 2-2 Pade log-determinant (Eq. 9-10, 16)
 * plus an SLQ estimate from the same CG coefficients, the 2p+1 finite-difference gradient
 * (Eq. 11) and Algorithm 1.
 *
 * Conventions (apply to every call unless stated otherwise)
 *  - Pointers are DEVICE pointers on the context's device unless marked [host].  Inputs
 *    marked [host|device] may be either; host buffers are staged through the workspace
 *    (that copy is part of the call).  Arrays are contiguous, FP64, row-major, 8-byte
 *    aligned; clusters are contiguous: rows [offsets[i], offsets[i+1]) belong to cluster i
 *    ("partitioned into n_c clusters"; uneven sizes allowed, reading X4/P19).
 *  - Ownership: the caller owns every array and the single workspace buffer (allocate
 *    nugpr_workspace_size() bytes, e.g. a torch uint8 tensor).  Handles (nugpr_ctx,
 *    nugpr_blocks) are small host objects; a blocks handle points into the workspace and
 *    must be destroyed before the workspace is freed.  The library never calls cudaMalloc.
 *  - Streams: all device work is enqueued on the context stream.  Calls with [host]
 *    outputs synchronise that stream before returning; nugpr_build_blocks does too (it
 *    reads back the per-block factorisation status for the jitter ladder).
 *  - Errors: every call returns nugpr_status; nugpr_last_error() gives a thread-local
 *    message for the last failing call.  No call aborts the process.
 *  - Determinism: identical inputs give bit-identical outputs (fixed-order reductions,
 *    no floating-point atomics).
 */
#ifndef NUGPR_H
#define NUGPR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Exported symbols keep default visibility even when the library is built with
 * -fvisibility=hidden. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define NUGPR_MAX_PROBES 15   /* columns per apply = 1 (y) + m probes <= 16 */
#define NUGPR_NUM_EVALS 7     /* 2p+1 with p = 3 hyperparameters */

typedef enum {
  NUGPR_OK = 0,
  NUGPR_ERR_INVALID_ARG = 1,      /* theta <= 0, d < 1, bad enum, NULL pointer, misalignment */
  NUGPR_ERR_SHAPE = 2,            /* offsets not strictly increasing / offsets[0]!=0 / offsets[n_c]!=n, block too large */
  NUGPR_ERR_NOT_SPD = 3,          /* a diagonal block failed Cholesky after the jitter ladder */
  NUGPR_ERR_DEGENERATE_REPS = 4,  /* lambda_0 = lambda_min(K_rep) <= 0 (Eq. 26 needs lambda_0 > 0) */
  NUGPR_ERR_CG_NOT_CONVERGED = 5, /* cg_max_iter reached ("flag any instances"); outputs hold the last iterate */
  NUGPR_ERR_WORKSPACE = 6,        /* workspace too small */
  NUGPR_ERR_CUDA = 7,
  NUGPR_ERR_COMM = 8,             /* the allgather callback failed */
  NUGPR_ERR_INTERNAL = 9,         /* e.g. the lambda_0 Lanczos did not converge within its iteration cap */
  NUGPR_ERR_UNSUPPORTED = 10,
  NUGPR_ERR_BREAKDOWN = 11        /* a CG quantity went non-finite or p^T q <= 0 (non-finite inputs, or the
                                     operator is not SPD at this theta); the record holds the state reached */
} nugpr_status;

typedef enum {
  NUGPR_RBF = 0,            /* alpha*exp(-||x-x'||^2/(2 lambda^2)) — Eq. 2 with the square (reading X3/P1) */
  NUGPR_MATERN52 = 1,       /* alpha*(1+sqrt5 r/l+5r^2/(3l^2))exp(-sqrt5 r/l) (config C4) */
  NUGPR_RBF_AS_PRINTED = 2  /* Eq. 2 literally: alpha*exp(-||x-x'||_2/(2 lambda^2)) */
} nugpr_kernel;

/* PADE: Eq. (16) (Pade on Q(A)^{-1} z, literal P(A)); SLQ: Lanczos on Q(A) from the same CG's
 * coefficients (reading X1).  MBCG: ONE batched CG on A with [c, Z]
 * (1 apply per iteration), log-det by SLQ with f = log on A's own Lanczos tridiagonal;
 * logdet_pade is NaN in that mode. */
typedef enum { NUGPR_LOGDET_PADE = 0, NUGPR_LOGDET_SLQ = 1, NUGPR_LOGDET_MBCG = 2 } nugpr_logdet_mode;
/* Storage of the blocks the apply streams (reading X6): FP64 (the parity path, 1e-6), or an FP32
 * copy of H / G(lambda') read by the FP64-accumulating DMMA apply (half the HBM bytes of the
 * dominant kernel; 1e-3 bar).  FP32 needs the m = 8 DMMA path and clusters <= 512 points. */
typedef enum { NUGPR_BLOCKS_F64 = 0, NUGPR_BLOCKS_F32 = 1 } nugpr_block_storage;
typedef enum { NUGPR_GRAD_CENTRAL = 0, NUGPR_GRAD_FORWARD_HALVING = 1 } nugpr_grad_mode;
typedef enum { NUGPR_REP_GIVEN = 0, NUGPR_REP_CENTROID = 1, NUGPR_REP_MEDOID = 2 } nugpr_rep_mode;

/* Operator mode chosen by comparing theta with the theta_0 the blocks were built at
 * (Eq. 23-25). */
typedef enum { NUGPR_MODE_BASELINE = 0, NUGPR_MODE_NOISE = 1, NUGPR_MODE_SCALE = 2,
               NUGPR_MODE_GENERIC = 3 } nugpr_mode;

/* theta = (lambda, sigma^2, alpha); all > 0. */
typedef struct { double lengthscale, noise, outputscale; } nugpr_theta;

typedef struct {
  double cg_tol;               /* residual threshold on the split system, absolute (0.01) */
  int32_t cg_max_iter;         /* 2000 */
  int32_t num_probes;          /* m, Hutchinson vectors (8); 1..NUGPR_MAX_PROBES */
  uint64_t probe_seed;         /* splitmix64 counter stream (see synth.probes) when probes == NULL */
  const double* probes;        /* NULL, or device m x n matrix of +-1 in cluster-sorted order */
  const int32_t* replay_iters; /* [host] NULL, or 1+m iteration counts to run exactly (parity replay) */
  int32_t logdet_mode;         /* nugpr_logdet_mode used for L */
  int32_t block_storage;       /* nugpr_block_storage: storage of the streamed blocks H / G in the apply */
} nugpr_solve_cfg;

typedef struct {
  int32_t mode;                /* nugpr_grad_mode */
  int32_t max_halvings;        /* FORWARD_HALVING cap (20) */
  double step[3];              /* CENTRAL: relative h_i = step_i*theta_i (1e-3); HALVING: relative Delta_0 (0.1) */
  double threshold;            /* FORWARD_HALVING threshold (1e-3) */
  int32_t threshold_relative;  /* 1: |g-g_prev| < thr*max(1,|g|) (reading P13); 0: absolute (paper literal) */
  int32_t reserved;
} nugpr_grad_cfg;

/* One MLL evaluation record (Alg. 1 ComputeLoss). */
typedef struct {
  double L;            /* 1/2 (quad + logdet + n log 2pi), Eq. 3 */
  double quad;         /* y^T K''^{-1} y = c^T A^{-1} c, c = R^{-T} y */
  double logdet;       /* logdet_pade or logdet_slq per logdet_mode */
  double logdet_pade;  /* Eq. 16 with the Pade trace */
  double logdet_slq;   /* Eq. 16 with the SLQ trace from the Q(A)-CG coefficients */
  double logdet_R;     /* 2 sum log|R_i| */
  double lambda0;      /* lambda_min(K_rep(theta)) */
  double resid_y;      /* final ||r|| of the y column */
  double resid_q_max;  /* max final ||r|| over probe columns */
  int32_t iters_y;
  int32_t iters_q_max;
  int32_t iters_q[16];
  int32_t converged;   /* 1 if every column met cg_tol (or replay ran) and no breakdown occurred */
  int32_t mode;        /* nugpr_mode */
  int32_t breakdown;   /* 1 if a column hit a non-finite / non-positive CG quantity (status NUGPR_ERR_BREAKDOWN) */
  int32_t lanczos_iters;     /* Lanczos iterations of the lambda_0 this evaluation used (build's or its own) */
  int32_t lanczos_converged; /* 1 if that Lanczos met its Ritz-residual bound (else NUGPR_ERR_INTERNAL) */
  int32_t lambda0_degenerate;/* 1 if lambda_0 <= 1e-11 ||K_rep||_inf: not certifiably > 0 (DEGENERATE_REPS) */
  double probe_t[16];  /* Pade trace term t_j = z_j^T P(A) Q(A)^{-1} z_j of probe j (Eq. 10; j < m) */
  double probe_s[16];  /* SLQ term s_j ~ z_j^T log(A) z_j of probe j (from the CG coefficients; j < m) */
} nugpr_mll_out;

typedef struct nugpr_ctx nugpr_ctx;
typedef struct nugpr_blocks nugpr_blocks;

/* Allgather used for perturbation sharding across ranks: gathers `bytes` from every rank
 * into recv (world*bytes, rank order).  Returns 0 on success.  Supplied by the caller
 * (the Python binding routes it through torch.distributed, NCCL on GPU boxes). */
typedef int (*nugpr_allgather_fn)(const void* send, size_t bytes, void* recv, void* user);

/* PAR-2 ("at large n the clusters shard across GPUs as well, with an allreduce of
 * CG dot products"): FP64 sum-allreduce of `count` doubles, recv[k] = sum over ranks of send[k].
 * send / recv are DEVICE pointers into the workspace given to nugpr_build_blocks (never aliased),
 * enqueued in order on `stream` (the context's cudaStream_t); the call may return before the
 * data moved (NCCL) as long as later work on `stream` sees the result.  Returns 0 on success.
 * The library only reduces zero-padded per-cluster partial arrays: every rank writes the slots
 * of its own clusters and zeros elsewhere, so the sum is exact (x + 0 = x) and every rank gets
 * the same partials a single GPU would have produced, in the same order. */
typedef int (*nugpr_allreduce_fn)(const double* send, double* recv, size_t count, void* stream, void* user);

const char* nugpr_version(void);
const char* nugpr_last_error(void);

/* Context on `device`, enqueuing on `cuda_stream` (cudaStream_t; NULL = legacy default).
 * device < 0 creates a host-only context (no CUDA calls; rank/world/allgather only) usable with
 * the host helpers below (nugpr_numgrad_exchange). */
nugpr_status nugpr_ctx_create(int device, void* cuda_stream, int rank, int world, nugpr_ctx** out);
nugpr_status nugpr_ctx_set_allgather(nugpr_ctx* ctx, nugpr_allgather_fn fn, void* user);
/* PAR-2 cluster sharding on this context (fn != NULL enables it, NULL disables).  Then
 * nugpr_build_blocks keeps only this rank's contiguous cluster range (nugpr_shard_range) and every
 * later call on those blocks (mll, numgrad, train) is COLLECTIVE: all ranks call it with identical
 * arguments (global offsets, full X_sorted / reps / y_sorted) and receive identical results.
 * Per CG iteration the ranks exchange three partial arrays through `fn` (S(A p) of the low-rank
 * term, p^T q, and r^T r with S(r)); everything else (K_rep, lambda_0, M', the 3-scalar CG state)
 * is replicated.  Small-block layouts only (clusters <= 512 points); mll_exact / predict /
 * the mBCG log-det mode return NUGPR_ERR_UNSUPPORTED on sharded blocks.  world = 1 is allowed
 * (exercises the exchange path on one GPU).  Errors: every decision that ends a call early is
 * taken on replicated data (the CG state, lambda_0, the exchanged jitter-ladder outcome), so all
 * ranks return the same status together; only a failing callback (NUGPR_ERR_COMM) can leave the
 * other ranks inside an exchange — treat it as fatal for the process group. */
nugpr_status nugpr_ctx_set_cluster_shard(nugpr_ctx* ctx, nugpr_allreduce_fn fn, void* user);

/* In-library NCCL (the library owns its collectives; PyTorch only carries the id).
 * nugpr_nccl_unique_id writes an ncclUniqueId (NUGPR_NCCL_ID_BYTES bytes, caller memory) on ONE
 * rank; the caller broadcasts those bytes to every rank (any transport), and every rank calls
 * nugpr_ctx_set_nccl(ctx, id) — collective over the context's (rank, world), blocking until all
 * ranks joined.  From then on the context's exchanges run as NCCL collectives on the context
 * stream instead of the callbacks: the PAR-1 record allgather (through a 64 KB device scratch the
 * call allocates — the library's only own device allocation, freed by nugpr_ctx_destroy) and the
 * PAR-2 partial allreduces (FP64 sum on workspace pointers), which are then captured into the
 * evaluation's device-driven CUDA graph (no host round trip per CG iteration).  NCCL is resolved
 * at run time from the libnccl.so.2 already mapped into the process (torch's), else the loader
 * path.  Errors: UNSUPPORTED (no libnccl), COMM (NCCL error; fatal for the group), CUDA. */
#define NUGPR_NCCL_ID_BYTES 128
nugpr_status nugpr_nccl_unique_id(uint8_t* id);
nugpr_status nugpr_ctx_set_nccl(nugpr_ctx* ctx, const uint8_t* id);
/* 1 if the context's sharded evaluations run their CG loop as a captured graph with the NCCL
 * exchanges inside (0: host-driven loop — callbacks, profiling, graphs off, or the capture of the
 * collectives was refused by the driver, after which the library keeps the host-driven loop). */
int32_t nugpr_ctx_sharded_graphs(const nugpr_ctx* ctx);
nugpr_status nugpr_ctx_destroy(nugpr_ctx* ctx);

/* Execution options of a context (defaults in brackets).
 *  NUGPR_OPT_SHARD_CLUSTERS [0]: 1 enables PAR-2 cluster sharding (as nugpr_ctx_set_cluster_shard)
 *    over the in-library NCCL communicator (or the allreduce callback if one is set).
 *  NUGPR_OPT_GRAPHS [1]: each evaluation's CG loop runs as ONE CUDA graph whose conditional WHILE node
 *    is driven by the device (no host round trip per iteration); 0: the same kernels launched directly
 *    with a host poll of the activity flag every 4 iterations (profiling with ncu, which cannot see
 *    kernels inside conditional graphs).  Both give bit-identical results. */
typedef enum { NUGPR_OPT_GRAPHS = 0, NUGPR_OPT_SHARD_CLUSTERS = 1 } nugpr_option;
nugpr_status nugpr_ctx_set_option(nugpr_ctx* ctx, int32_t option, int32_t value);

/* Kernel-class profiler (bench.py's live roofline): when enabled, CUDA events are recorded on
 * the context stream around every launch of a class; accumulators reset on (re-)enable.
 * cls: 0 apply with a block term (noise/scale/generic), 1 apply without (baseline), 2 CG update,
 *      3 rhs/init, 4 block GEMMs (H, G), 5 Cholesky+inverse, 6 Lanczos lambda_0, 7 other.
 * ms: summed event time; bytes: summed ALGORITHMIC bytes (apply classes only: 8*(sum b_i^2 +
 * 2 n c + n + n_c^2) per launch with a block term, 8*(2 n c + n + n_c^2) without);
 * launches: number of timed launches. */
nugpr_status nugpr_ctx_set_profiling(nugpr_ctx* ctx, int32_t enable);
nugpr_status nugpr_ctx_profile(nugpr_ctx* ctx, int32_t cls, double* ms, double* bytes, int64_t* launches);
/* Total kernel launches issued by the library in this process. */
int64_t nugpr_launch_count(void);

/* A0 — clustering ("k-means to find n_c clusters", cluster centres become the
 * representatives; PAPER.md:43, 290 cluster-contiguous storage; Eq. (32)
 * medoids).  Lloyd k-means per reading P18: squared distances summed in dimension order
 * without FMA, ties to the lowest centre, centroid sums exact in int64 fixed point at scale
 * 2^s with s = 62 - ceil(log2(max|x| n)), empty clusters keep their centre; stop when no
 * assignment changes or after max_iter update steps.  Then a stable sort by (cluster,
 * original index).  The assignment, perm and offsets are bit-exact functions of the inputs.
 *  X [host|device] n x d original order (d <= 32).  init_centers [host|device] n_c x d, or NULL
 *  for Forgy rows x_{i_j}: candidate t of centre j is splitmix64_seed((j<<32)|t) mod n, the first
 *  not yet taken.  rep_mode nugpr_rep_mode: GIVEN = the initial centres, CENTROID = the final
 *  centres, MEDOID = argmax_{x in C_j} sum_{x' in C_j} k(x, x'; theta) (reading P17; `kernel`,
 *  theta.lengthscale/outputscale used only here), lowest original index on ties.
 *  y [host|device] n or NULL.  Outputs (each [host|device], NULL to skip except offsets):
 *  perm n (perm[k] = original row of sorted row k), offsets [host] n_c+1, reps n_c x d,
 *  X_sorted n x d, y_sorted n, iters [host] (update steps made).  An empty final cluster
 *  returns NUGPR_ERR_SHAPE (outputs are still written).  workspace: nugpr_cluster_workspace_size. */
nugpr_status nugpr_cluster_workspace_size(int64_t n, int32_t d, int32_t n_c, size_t* bytes);
nugpr_status nugpr_cluster(nugpr_ctx* ctx, const double* X, int64_t n, int32_t d, int32_t n_c,
                           const double* init_centers, uint64_t seed, int32_t max_iter,
                           int32_t rep_mode, int32_t kernel, nugpr_theta theta, const double* y,
                           void* workspace, size_t ws_bytes, int64_t* perm, int64_t* offsets,
                           double* reps, double* X_sorted, double* y_sorted, int32_t* iters);

/* Workspace bytes for blocks built on `offsets` ([host], n_c+1) plus `eval_slots` (1..7)
 * evaluation scratch sets (up to NUGPR_MAX_PROBES probes, cg_max_iter < 4096).  More slots
 * let nugpr_numgrad keep several evaluations in flight; nugpr_build_blocks uses as many as
 * fit in the bytes it is given. */
nugpr_status nugpr_workspace_size(const int64_t* offsets, int32_t n_c, int32_t d,
                                  int32_t eval_slots, size_t* bytes);
/* PAR-2: the contiguous cluster range [range[0], range[1]) rank `rank` of `world` owns, balanced
 * by the streamed block bytes sum_i ld_i^2 (ld_i = b_i rounded up to 8), at least one cluster per
 * rank (n_c >= world, else NUGPR_ERR_SHAPE); and the workspace bytes of that rank's blocks
 * (eval_slots as above; global offsets).  Host-only. */
nugpr_status nugpr_shard_range(const int64_t* offsets, int32_t n_c, int32_t rank, int32_t world, int32_t range[2]);
nugpr_status nugpr_workspace_size_shard(const int64_t* offsets, int32_t n_c, int32_t d, int32_t eval_slots,
                                        int32_t rank, int32_t world, size_t* bytes);

/* A1 — Alg. 1 line 264 at theta0: K_i assembled on the fly from X_sorted, R_i = chol(K_i)
 * with the jitter ladder, logdet_R, u_i = R_i^{-T} 1, H_i = R_i^{-T} R_i^{-1}, K_rep,
 * lambda_0, M = K_rep - lambda_0 I.
 *  X_sorted [host|device] n x d, offsets [host] n_c+1, reps [host|device] n_c x d.
 *  failed_block [host]: -1, or the block index on NUGPR_ERR_NOT_SPD.
 *  max_jitter [host]: largest jitter added (0 if none). */
nugpr_status nugpr_build_blocks(nugpr_ctx* ctx, const double* X_sorted, const int64_t* offsets,
                                int32_t n_c, int32_t d, const double* reps, int32_t kernel,
                                nugpr_theta theta0, void* workspace, size_t ws_bytes,
                                nugpr_blocks** out, int32_t* failed_block, double* max_jitter);
nugpr_status nugpr_blocks_destroy(nugpr_blocks* blocks);

/* Debug read-back of block data into a [host] buffer of `bytes` (tests only).
 *  what: 0 Linv (packed per block as ld_i x ld_i col-major, padded), 1 H (same layout),
 *        2 u (n, cluster-sorted order), 3 jitter (n_c), 4 scalars {logdet_R, lambda0},
 *        5 M (n_c x n_c), 6 ld (int32 n_c), 7 the probe matrix generated for seed/num_probes
 *        of the last nugpr_mll call (m x n). */
nugpr_status nugpr_blocks_export(const nugpr_blocks* blocks, int32_t what, void* dst, size_t bytes);

/* A2-A7 — one MLL evaluation (Alg. 1 ComputeLoss) at theta with the blocks built at theta0.
 *  y_sorted [host|device] n.  out [host]. */
nugpr_status nugpr_mll(nugpr_ctx* ctx, nugpr_blocks* blocks, const double* y_sorted,
                       nugpr_theta theta, const nugpr_solve_cfg* cfg, nugpr_mll_out* out);

/* A8 — numerical gradient at theta (= the blocks' theta0).  CENTRAL: 7 evaluations
 * theta, theta +- h_i e_i, g_i = (L+ - L-)/(2 h_i), sharded over the context's ranks
 * (perturbation parallel; results exchanged with the allgather callback).
 * FORWARD_HALVING: Alg. 1 lines 266-278 (rank-local).  evals [host]: NULL or room for
 * max(7, 1+3*(max_halvings+1)) records; n_evals [host]: number written. */
nugpr_status nugpr_numgrad(nugpr_ctx* ctx, nugpr_blocks* blocks, const double* y_sorted,
                           nugpr_theta theta, const nugpr_grad_cfg* gcfg,
                           const nugpr_solve_cfg* scfg, double* L0, double grad[3],
                           nugpr_mll_out* evals, int32_t* n_evals);

/* A9 — Algorithm 1: for each epoch build blocks at theta, numgrad, Adam (gamma = lr,
 * beta = (0.9, 0.999), eps = 1e-8, theta clamped >= 1e-8).
 *  adam_state [host] in/out: theta[3], m[3], v[3], t (10 doubles); resumable.
 *  records [host] epochs x NUGPR_TRAIN_RECORD doubles:
 *    {L0, g[3], theta[3] (before the step), iters_y_max, iters_q_max, jitter, n_evals, reserved} */
#define NUGPR_TRAIN_RECORD 12
nugpr_status nugpr_train(nugpr_ctx* ctx, const double* X_sorted, const int64_t* offsets,
                         int32_t n_c, int32_t d, const double* reps, const double* y_sorted,
                         int32_t kernel, int32_t epochs, double lr, const nugpr_grad_cfg* gcfg,
                         const nugpr_solve_cfg* scfg, double adam_state[10], double* records,
                         void* workspace, size_t ws_bytes);

/* NEXT-2 — the EXACT structured MLL at the blocks' theta_0, from the
 * structure of Eq. (28)-(29) with no probes, Pade or CG: W = R^{-T}E has
 * disjoint columns u_i, D = diag(u_i^T u_i), M~ = D^{1/2} M D^{1/2}, C = I + M~ = L_C L_C^T,
 * c = R^{-T} y, zeta_i = u_i^T c_i / sqrt(d_i):
 *     log|K''| = logdet_R + log|C|                                  (matrix determinant lemma)
 *     y^T K''^{-1} y = c^T c - (zeta^T zeta - ||L_C^{-1} zeta||^2)  (Woodbury, M~ C^{-1} = I - C^{-1})
 *     L = (quad + log|K''| + n log 2 pi) / 2.
 *  y_sorted [host|device] n.  out [host] 4 doubles: {L, quad, logdet, log|C|}.
 *  Uses the blocks' first evaluation slot as scratch (same n_c bound as nugpr_predict).
 *  NUGPR_ERR_NOT_SPD if C is not SPD (lambda_0 did not make M PSD). */
nugpr_status nugpr_mll_exact(nugpr_ctx* ctx, nugpr_blocks* blocks, const double* y_sorted, double out[4]);

/* NEXT-1 — posterior at the blocks' theta_0 (build the blocks at the trained theta): Eq. (4)-(5)
 * (PAPER.md:68-73), mean = K*^T K''^{-1} y, var = alpha - diag(K*^T K''^{-1} K*) (+ sigma^2 when
 * add_noise; reading P22), with K* = k(X_train, X_test) generated on the fly and K''^{-1} applied
 * EXACTLY through the Woodbury form of Eq. (28) (no CG; oracle/predict.py gives the algebra).
 *  y_sorted [host|device] n; X_test [host|device] n_test x d; mean [host|device] n_test;
 *  var [host|device] n_test or NULL.  Uses the blocks' first evaluation slot as scratch.
 *  Any n_c whose (n_c rounded up to 8)^2 doubles fit in one slot vector (16 n_pad doubles; else
 *  NUGPR_ERR_WORKSPACE); n_c > 512 factorises I + M~ with the blocked big-block kernels. */
nugpr_status nugpr_predict(nugpr_ctx* ctx, nugpr_blocks* blocks, const double* y_sorted, const double* X_test,
                           int64_t n_test, int32_t add_noise, double* mean, double* var);

/* Host-only helpers (no device work; usable without a GPU). */
/* PAR-1 exchange of nugpr_numgrad CENTRAL: the 7 evaluations theta, theta +- h_i e_i
 * (h_i = step_i theta_i) are owned per nugpr_shard_plan(world, {1,3,3,2,2,2,2}); this rank passes
 * the losses of the evaluations it owns in L_mine[k] (others ignored) and their statuses in
 * status_mine[k] ([host] or NULL = all OK); one allgather through the context callback; every rank
 * returns the same L0 = L(theta) and g_i = (L+ - L-)/(2 h_i) (Eq. 11 as a central difference,
 * reading X2) and the same status: the first failed evaluation's (hard failures before
 * NUGPR_ERR_CG_NOT_CONVERGED).  nugpr_numgrad uses the same exchange and ALWAYS reaches it, failed
 * evaluations included, so one rank's failure never leaves the others waiting in the allgather. */
nugpr_status nugpr_numgrad_exchange(nugpr_ctx* ctx, nugpr_theta theta, const double step[3],
                                    const double L_mine[7], const int32_t* status_mine, double* L0,
                                    double grad[3]);
/* One Adam step on state {theta[3], m[3], v[3], t}. */
nugpr_status nugpr_adam_step(double state[10], const double grad[3], double lr);
/* Longest-processing-time assignment of n tasks with costs to `world` ranks: owner[n]. */
nugpr_status nugpr_shard_plan(int32_t world, const double* costs, int32_t n, int32_t* owner);
/* Symmetric tridiagonal eigen-decomposition (implicit QL) returning eigenvalues and first
 * eigenvector components; the SLQ kernel's routine, exported for host-side tests. */
nugpr_status nugpr_tridiag_eig(int32_t k, const double* diag, const double* off,
                               double* evals, double* first);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* NUGPR_H */
