// kernels_decl.h — host-side launchers of the nuGPR kernels (internal).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nugpr.h"
#include "common.cuh"

namespace nugpr {

// Count of kernel launches issued by this library (bench.py reports it as gpu_launches).
void note_launch(long long n = 1);
long long launch_count();
// Opt a kernel into the largest dynamic shared memory the device allows (optin limit minus the
// kernel's static shared memory); cached per function.
void smem_optin(const void* func);
// NUGPR_DEBUG_SYNC=1: synchronise and report after every launch (debugging only).
void post_launch(const char* name);

// build_kernels.cu
void launch_assemble(const double* X, int d, const LayoutDev& L, const int32_t* list, int nlist,
                     int ld_max, const double* jitter, double* dst, int kind, double lam,
                     double noise, double alpha, cudaStream_t s);
size_t chol_smem_bytes(int ld_max);
void launch_chol_trtri(double* A, const LayoutDev& L, const int32_t* list, int nlist, int ld_max,
                       int32_t* status, double* logdet_blk, double* u, cudaStream_t s);
// H = Linv Linv^T and G = Linv T: packed output (PACKED storage at L.pboff) for the small layout,
// full ld x ld storage at L.boff for the big-block layout
void launch_gemm_H(const double* Linv, double* H, const LayoutDev& L, int ld_max, bool packed, cudaStream_t s);
void launch_gemm_KLt(const double* K, const double* Linv, double* T, const LayoutDev& L, int ld_max,
                     cudaStream_t s);
void launch_gemm_LT(const double* Linv, const double* T, double* G, const LayoutDev& L, int ld_max, bool packed,
                    cudaStream_t s);
void launch_sum(const double* v, int n, double* out, cudaStream_t s);
void launch_krep(const double* reps, int n_c, int d, int kind, double lam, double alpha, double* K,
                 cudaStream_t s);
size_t lanczos_scratch_doubles(int n_c, int kmax);
// Returns the launch status (a cluster launch can fail for lack of shared memory / co-residency).
cudaError_t launch_lanczos(const double* K, int n_c, const double* vinit, double* scratch, int kmax,
                           double tol_rel, double* lam0, double* v0, double* M, int32_t* info,
                           cudaStream_t s);

// eval_kernels.cu
void launch_apply(const ApplyArgs& a, int ncp, cudaStream_t s);
void launch_update(const UpdateArgs& a, int ncp, cudaStream_t s);
void launch_lowrank(const LowrankArgs& a, int ncp, cudaStream_t s);
void launch_rhs_init(const RhsArgs& a, int ld_max, cudaStream_t s);
void launch_cy(const LayoutDev& L, const double* Linv, const double* y, int ld_max, double* cy, cudaStream_t s);
int num_sms_host();
void launch_d2f(const double* src, float* dst, int64_t n, cudaStream_t s);
void launch_spart(const LayoutDev& L, const double* u, const double* V, int ncol, double* part,
                  cudaStream_t s);
void launch_final(const CGState* st, const EvalParams* prm, const double* ah, const double* bh,
                  int stride, double* slq_work, const double* logdet_R, double n,
                  int ncol, int logdet_mode, nugpr_mll_out* out, cudaStream_t s,
                  const double* quad_part = nullptr, int n_quad_part = 0);
// PAR-2: single-CTA CG finaliser (FIN_INIT / FIN_ALPHA / FIN_UPDATE / FIN_TRACE) over exchanged partials
void launch_fin(int fin, CGState* st, const EvalParams* prm, const double* part, int n_tiles, int ncol,
                double* hist, int hist_stride, cudaStream_t s, const double* SR = nullptr, double* SP0 = nullptr,
                double* SP1 = nullptr, unsigned long long cond = 0);
int quad_parts(int64_t n_pad, int cap);
void launch_quad_part(const double* c, const double* x, int64_t n_pad, int nparts, double* part, cudaStream_t s);
void launch_probe_gen(uint64_t seed, int m, int64_t n, double* Z, cudaStream_t s);

// apply_kernels.cu (packed symmetric blocks, ld_max <= 512)
// Plans the launch (smem ring, m-tiles per warp, probe n-tiles) into a; false if it cannot run.
bool plan_packed_apply(int ld_max, int ncol, bool f32, int seg_max, int lr_nc, ApplyArgs& a);
void launch_apply_packed(const ApplyArgs& a, cudaStream_t s);

// big_kernels.cu (ld_max > 512)
size_t big_scratch_doubles(int n_c, int ld_max);
void launch_big_chol_trtri(double* A, const LayoutDev& L, const int32_t* list, int nlist, int ld_max,
                           int32_t* status, double* logdet_blk, double* u, double* scratch, cudaStream_t s);
void launch_apply_big(const ApplyArgs& a, int ncp, cudaStream_t s);

// predict_kernels.cu (NEXT-1)
void launch_pred_ks(const double* X, const double* Xt, int d, const LayoutDev& L, int nt, int ld_max, int kind,
                    double lam, double alpha, double* Ks, cudaStream_t s);
void launch_pred_trmm(const double* Lm, const double* Bm, double* Cm, const int32_t* ld, const int64_t* loff,
                      const int64_t* goff, int groups, int nt, int ld_max, cudaStream_t s);
void launch_pred_reduce(const LayoutDev& L, const double* W, const double* c, const double* u, int nt, double* wc,
                        double* ww, double* p, cudaStream_t s);
void launch_exact_final(const LayoutDev& L, const double* c, const double* zeta, const double* lz,
                        const double* logdet_R, const double* logdet_C, double* ccblk, int64_t n, double* out,
                        cudaStream_t s);
void launch_pred_setup(const LayoutDev& L, const double* c, const double* u, const double* M, int ldc, double* zeta,
                       double* sd, double* Cm, cudaStream_t s);
void launch_pred_lz(const double* Lc, int ldc, int n_c, const double* zeta, double* lz, cudaStream_t s);
void launch_pred_pcol(const double* p, int n_c, int nt, int ldc, double* pc, cudaStream_t s);
void launch_pred_final(int n_c, int nt, int ldc, const double* wc, const double* ww, const double* p, const double* lp,
                       const double* zeta, const double* lz, double alpha, double noise_add, double* mean, double* var,
                       int64_t mean_off, int64_t var_off, cudaStream_t s);

// cluster_kernels.cu (row A0)
void launch_km_absmax(const double* X, int64_t cnt, unsigned long long* out, cudaStream_t s);
size_t km_assign_smem();
void launch_km_assign(const double* X, int64_t n, int d, int n_c, const double* C, const int32_t* a_old,
                      int32_t* a_new, double scale, unsigned long long* S, unsigned long long* cnt,
                      int32_t* changed, cudaStream_t s);
void launch_km_update(int n_c, int d, double inv_scale, unsigned long long* S, unsigned long long* cnt,
                      double* C, cudaStream_t s);
int64_t km_chunks(int64_t n);
void launch_km_sort(const int32_t* a, int64_t n, int n_c, long long* hist, int64_t* perm, int64_t* off,
                    cudaStream_t s);
void launch_km_gather(const double* src, int width, const int64_t* idx64, const int32_t* idx32, int64_t rows,
                      double* dst, cudaStream_t s);
void launch_km_medoids(const double* Xs, int d, const int64_t* off, int n_c, int64_t b_max, int kind, double lam,
                       double alpha, double* score, int64_t* out, cudaStream_t s);

}  // namespace nugpr
