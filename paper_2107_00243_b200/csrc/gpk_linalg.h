// Launchers for the mBCG vector kernels, Woodbury GEMMs and pivoted Cholesky.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace gpk {

enum { kFlagConverged = 1, kFlagError = 2 };
enum { kStatusOk = 0, kStatusAlpha = 1, kStatusRz = 2 };

// Per-column CG scalars (krylov.hpp:66-68), resident on the device.
struct SlotState {
  double rz, norm0, alpha, beta, alpha_prev, beta_prev, bad;
  double pres;  // last recorded preconditioned residual norm ||P^-1 r_k|| (krylov.hpp:102)
  int col, iters, status, flag;
};

int num_chunks(int n);
cudaError_t launch_dot_partials(int op, const double* A, const double* B, double sig2, int n, long long ldn, int t,
                                double* part, cudaStream_t st);
cudaError_t launch_reduce_partials(const double* part, int nrb, int t, double* out, cudaStream_t st);
cudaError_t launch_cg_init(const double* part_rz, const double* part_zz, int nrb, int t, SlotState* ss,
                           cudaStream_t st);
cudaError_t launch_cg_alpha(const double* part, int nrb, int t, int k, SlotState* ss, double* alpha_hist,
                            int max_iters, cudaStream_t st);
cudaError_t launch_cg_beta(const double* part_rz, const double* part_zz, int nrb, int t, int k, double rel_tol,
                           SlotState* ss, double* beta_hist, double* resid_hist, int max_iters, cudaStream_t st);
cudaError_t launch_cg_update_xr(double* X, double* R, const double* P, const double* Y, double sig2, int n,
                                long long ldn, int t, const SlotState* ss, cudaStream_t st);
cudaError_t launch_cg_update_p(double* P, const double* Z, int n, long long ldn, int t, const SlotState* ss,
                               cudaStream_t st);
cudaError_t launch_gather_cols(const double* src, long long lds, const int* map, double scale, int n, int t,
                               double* dst, long long ldd, cudaStream_t st);
cudaError_t launch_scatter_cols(const double* src, long long lds, const int* map, int n, int t, double* dst,
                                long long ldd, cudaStream_t st);
cudaError_t launch_axpby(double* a, const double* b, double alpha, double beta, int n, int t, long long ld,
                         cudaStream_t st);
cudaError_t launch_woodbury_finish(const double* R, const double* T, double sig2, int n, long long ldn, int t,
                                   double* Z, cudaStream_t st);

size_t g1_workspace(int n, int ka, int tb);
cudaError_t launch_g1(const double* A, long long lda, int ka, const double* B, long long ldb, int tb, int n,
                      double* part, double* W, long long ldw, cudaStream_t st);
cudaError_t launch_g2(const double* A, long long lda, int ka, const double* W, long long ldw, int tb, int n,
                      double* T, long long ldt, cudaStream_t st);
// Z = R / s2 - (C W) / s2 (G2 fused with the Woodbury finish, preconditioners.hpp:114-118)
cudaError_t launch_woodbury_apply(const double* C, long long ldc, int ka, const double* W, long long ldw,
                                  const double* R, long long ldr, double sig2, int tb, int n, double* Z,
                                  long long ldz, cudaStream_t st);

// gpk_cgfused.cu: the fused single-rank CG iteration (see the file header)
int g1_chunk_rows(int n, int ka = 0);
cudaError_t launch_g1_reduce(const double* part, int n, int ka, int tb, double* W, long long ldw, cudaStream_t st);
int g2_row_blocks(int n);
// vmax (nullable): cleared per column by the last CTA (the |p| maxima of this iteration's p
// update are accumulated into it afterwards)
cudaError_t launch_cg_pap_alpha(const double* P, double* Y, double sig2, int n, long long ldn, int t,
                                double* part, unsigned* cnt, int k, SlotState* ss, double* alpha_hist, int max_iters,
                                cudaStream_t st, unsigned long long* vmax = nullptr, const double* parts = nullptr,
                                int splits = 0, long long sstride = 0, long long ldp = 0);
cudaError_t launch_g1_xr(const double* L, long long ldl, int ka, double* X, const double* R, double* Rn,
                         const double* P, const double* Y, double sig2, long long ldn, int tb, int n,
                         const SlotState* ss, double* part, double* W, long long ldw, cudaStream_t st);
cudaError_t launch_g2_dots_beta(const double* C, long long ldc, int ka, const double* W, long long ldw, int tb, int n,
                                double* Z, const double* R, long long ldn, double sig2, double* prz, double* pzz,
                                unsigned* cnt, int k, double rel_tol, SlotState* ss, double* beta_hist,
                                double* resid_hist, int max_iters, unsigned long long* vmax, cudaStream_t st);
cudaError_t launch_cg_p_vmax(double* P, const double* Z, int n, long long ldn, int t, const SlotState* ss,
                             unsigned long long* vmax, cudaStream_t st);

// gpk_wood.cu: shared-memory-staged Woodbury GEMMs of the fused iteration (grid = 2 x SMs)
int wood_grid();
size_t wood_g1_workspace(int ka, int tb);
size_t wood_g2_partials(int tb);
// the whole single-rank CG vector phase of one iteration in ONE cooperative launch (gpk_wood.cu)
bool cg_iter_coop_available();
cudaError_t launch_cg_iter_coop(const double* L, long long ldl, const double* Cm, long long ldc, int ka, double* X,
                                double* R, double* P, double* Z, const double* Y, long long ldn, int tb, int n,
                                double sig2, double psig2, double* ppap, double* pg1, double* W, double* prz,
                                double* pzz, SlotState* ss, int k, double rel_tol, double* ahist, double* bhist,
                                double* rhist, int max_iters, unsigned long long* vmax, SlotState* snap,
                                cudaStream_t st);
// W = A^T R_new (A: ka columns, ld lda); with X != null, R_new = R - alpha (Y + s2 P) for live
// slots is written back to R and X += alpha P (krylov.hpp:94-95)
cudaError_t launch_g1s(const double* A, long long lda, int ka, double* R, long long ldr, int tb, int n,
                       double* part, double* W, long long ldw, double* X, const double* P, const double* Y,
                       double sig2, const SlotState* ss, cudaStream_t st);
// Z = (R - C W) / s2 with per-CTA r.z / z.z partials (prz, pzz: [tb][wood_grid()])
cudaError_t launch_g2s_dots_beta(const double* C, long long ldc, int ka, const double* W, long long ldw, int tb,
                                 int n, double* Z, const double* R, long long ldn, double sig2, double* prz,
                                 double* pzz, cudaStream_t st);
// beta_step from the G2s partials + p = z + beta p + |p| column maxima (vmax pre-cleared);
// cnt: t zeroed counters (re-armed by the kernel); snap (nullable, pinned host memory): a
// copy of the updated slot states for the host's pipelined read-back
cudaError_t launch_cg_beta_p(double* P, const double* Z, int n, long long ldn, int t, SlotState* ss,
                             const double* prz, const double* pzz, unsigned* cnt, int k, double rel_tol,
                             double* beta_hist, double* resid_hist, int max_iters, unsigned long long* vmax,
                             SlotState* snap, cudaStream_t st);

int pchol_blocks(int n);
struct PivotState {
  double dp;        // remaining diagonal at the current pivot
  long long p;      // current pivot
  int stopped;      // a stopping rule fired
  int negative;     // ... because of a negative pivot
  int done;         // steps completed
  int pad;
};
cudaError_t launch_pchol_dev(int family, const double* sx, const double* sq, int n, int d, double o2, double* L,
                             int rank, double diag_tol, double kmax, double* col, double* dg, double* bval,
                             long long* bidx, PivotState* ps, long long* pivots, cudaStream_t st);
// gpk_pchol.cu: the whole pivoted Cholesky in one cooperative launch (grid = pchol_persistent_grid;
// cval / cidx hold 2 * grid candidates), and the blocked derivative-factor kernels.
int pchol_persistent_grid(int n, size_t smem);
cudaError_t launch_pchol_persistent(int family, const double* sx, const double* sq, int n, int d, double o2,
                                    double* L, int rank, double diag_tol, double kmax, double* dg, double* cval,
                                    long long* cidx, PivotState* ps, long long* pivots, int grid, cudaStream_t st);
// row-sharded pivoted Cholesky (gpk_pchol.cu): per-step kernels on the own rows, candidates and
// the pivot row exchanged by all-gathers between them
int pchol_shard_grid(int nl);
cudaError_t launch_pchol_shard_step(int family, const double* sx, const double* sq, int n, int d, double o2,
                                    double* L, long long ldl, int r0, int nl, int s, const double* lp,
                                    const PivotState* ps, double* dg, double* cval, long long* cidx, int grid,
                                    double* send, cudaStream_t st);
cudaError_t launch_pchol_shard_select(const double* cand, int world, int s, double diag_tol, double kmax,
                                      PivotState* ps, long long* pivots, const double* L, long long ldl, int r0,
                                      int nl, int k, double* rowsend, cudaStream_t st);
cudaError_t launch_pchol_shard_rowtake(const double* recv, int world, int k, const int* rr0, const int* rrows,
                                       const PivotState* ps, double* lp, cudaStream_t st);
cudaError_t launch_pchol_pivot_rows(int phase, const double* src, double* dst, long long ldl, int r0, int nl, int k,
                                    const long long* piv, int world, const int* rr0, const int* rrows,
                                    cudaStream_t st);
cudaError_t launch_gather_ext_rows(const double* src, long long lds, int cols, int r0, int nl, const long long* piv,
                                   int k, double* dst, long long ne, cudaStream_t st);
cudaError_t launch_iota_ll(long long* out, int k, long long base, cudaStream_t st);
cudaError_t launch_deriv_columns_block(int family, const double* sx, const double* x, const double* sq, int n, int d,
                                       const long long* piv, int bb, int nw, const double* facs, double o2,
                                       double* DC, long long dcw_stride, cudaStream_t st);
size_t dl_replay_workspace(int nw);
cudaError_t launch_dl_block(const double* L, double* dL, long long wstride, int nw, int s0, int bb,
                            const long long* piv, const double* DC, long long dcw_stride, int n, double* rep,
                            cudaStream_t st);
cudaError_t launch_kernel_deriv_columns(int family, const double* sx, const double* x, const double* sq, int n, int d,
                                        long long p, int nw, const double* facs, double o2, double* out,
                                        cudaStream_t st);
cudaError_t launch_argmax(const double* v, int n, double* bval, long long* bidx, double* out_val,
                          long long* out_idx, cudaStream_t st);
cudaError_t launch_pchol_step(double* L, long long ldl, int s, long long p, double root, const double* col, double* dg,
                              int n, double* bval, long long* bidx, double* out_val, long long* out_idx,
                              cudaStream_t st);
cudaError_t launch_dl_inblock(const double* L, long long ldl, double* dL, long long wstride, int nw, int s0, int q,
                              long long p, const double* DC, long long dcw_stride, int n, cudaStream_t st);
cudaError_t launch_gather_pivot_rows(const double* M, long long ldm, long long mstride, int nw,
                                     const long long* piv, int s0, int b, double* out, cudaStream_t st);
cudaError_t launch_dl_step(const double* L, long long ldl, double* dL, long long wstride, int nw, int s, long long p,
                           const double* dcol, long long dcol_stride, int n, cudaStream_t st);

}  // namespace gpk
