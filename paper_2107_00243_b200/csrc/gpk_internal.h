// Internal launcher interface between the host driver and the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gpk {

enum { kRBF = 0, kMatern12 = 1, kMatern32 = 2, kMatern52 = 3 };
enum { kModeValue = 0, kModeDls = 1 };  // K entries / dK/dlengthscale_j entries

struct MvmArgs {
  int n;                     // rows/cols of K
  int n_pad;                 // padded to a multiple of 128
  int t;                     // active columns
  long long ldo;             // output leading dimension (column-major)
  int jdim;                  // lengthscale index for kModeDls
  int jtiles_per_split;      // j-tiles (of 32) handled by one split
  double scale;              // output scale (o^2, 2o, -2 o^2 / l_j / c_fam, ...)
  long long split_stride;    // element offset between split-K partial outputs
  int flush;                 // tcgen05 path: j-tiles per TMEM accumulation group (fp64 drain period)
  int row_begin;             // first output row of this rank's shard (multiple of 128)
  int row_end;               // one past the last output row; outputs are stored at row - row_begin
  int dp;                    // padded coordinate count of the packed fp32 rows (Gram guard path)
  int ctas;                  // tcg MVM: persistent grid size (0: one CTA per (row block, split) unit)
  int unit_order;            // tcg MVM, persistent grid: 0 = contiguous units per CTA, 1 = strided (all CTAs in one split)
};

// Packed-operand geometry for a given column count.
struct MvmShape {
  int tn;    // columns per thread (8 column groups)
  int vld;   // leading dimension (elements) of the packed V rows
  int cgs;   // column-group stride
};
MvmShape mvm_shape(int t, bool fp64, int mode);
int dpad_for(int d);  // padded dimension of the packed coordinates
// Scale applied to the scaled coordinates in FP32 mode: s' = c_fam * s.
double prescale_c(int family);

// Fused kernel MVM on packed operands: X [n_pad][DP], V [n_pad][vld] (mvm_shape layout).
// out: column-major [t][ldo] fp64 (split-K partials use split_stride, then reduced).
cudaError_t launch_fused_kmvm(bool fp64, int family, int dp, int mode, const void* X, const void* V,
                              double* out, const MvmArgs& a, int splits, cudaStream_t st);
// gpk_mvm_f64g.cu: fp64 value MVM on the fp64 tensor cores (reference expanded distances)
cudaError_t launch_fused_kmvm_f64g(int family, int dp, const double* X, const double* sq, int n, const double* V,
                                   long long ldv, int tc, double* out, long long ldo, double scale, int row_begin,
                                   int row_end, cudaStream_t st);
// gpk_probes.cu: n x count Rademacher probes +-1/sqrt(n) from one mt19937_64(seed) stream, column-major
cudaError_t launch_make_probes(long long n, int count, unsigned long long seed, double* out, cudaStream_t st);
cudaError_t launch_reduce_splits(const double* part, int splits, long long split_stride, int t, int n,
                                 long long ldpart, double* out, long long ldo, cudaStream_t st);

// Pack fp64 column-major X (n x d) into the scaled row-major MVM layouts.
cudaError_t launch_pack_x(const double* X, long long ldx, int n, int d, int n_pad, const double* ls,
                          double prescale, int dp32, float* X32, int dp64, double* X64s, double* sx_colmajor,
                          double* sqnorm, cudaStream_t st);
// Pack fp64 column-major V (t columns, ld) into the packed MVM layout; optional slot->column map.
cudaError_t launch_pack_v32(const double* V, long long ldv, const int* colmap, int t, int n, int n_pad,
                            MvmShape sh, float* V32, cudaStream_t st);
cudaError_t launch_pack_v64(const double* V, long long ldv, const int* colmap, int t, int n, int n_pad,
                            MvmShape sh, double* V64, cudaStream_t st);

// tcgen05 (tensor-core, 3xTF32) fused MVM: value mode, t <= 128 per launch.
int tc_npad(int t);  // padded column count (multiple of 8) of the packed V tiles, -1 if t > 128
cudaError_t launch_pack_v_tc(const double* V, long long ldv, int t, int n, int n_pad, int npad, float* vhi,
                             float* vlo, cudaStream_t st);
cudaError_t launch_fused_kmvm_tc(int family, int dp, const float* X, const float* vhi, const float* vlo, double* out,
                                 const MvmArgs& a, int splits, cudaStream_t st);

// Gram variant (both contractions on tcgen05): squared distances s_ij = n_i + n_j - 2 x~_i.x~_j
// straight out of a 3xTF32 MMA on augmented coordinates.  Packs x~ = (X / l - mean) pre-scaled
// as tf32 hi/lo 32x32 swizzled tiles: xh, xl hold 2 n_pad x 32 floats (the B-side image
// [x~, 1, n] then the A-side image [-2 x~, n, 1]); xn holds n_pad fp32 norms then n_pad / 64
// per-j-tile maxima; mu: d doubles of scratch.  RBF / Matern-3/2 / Matern-5/2, d <= 30.
constexpr int kGramMaxDim = 30;  // d + 2 augmented Gram coordinates in <= 32 tf32 columns
cudaError_t launch_gram_pack(const double* X, long long ldx, int n, int d, int n_pad, const double* ls,
                             double prescale, double* mu, float* xh, float* xl, float* xn, cudaStream_t st);
// V (t <= 96 columns) -> per-column power-of-two scaled fp16 hi/lo tiles (+ colscale_c =
// scale / (2^10 sigma_c) applied to the output); vmax: t uint64 scratch, colscale: t doubles.
int tcg_npad(int t);  // padded column count (multiple of 8, <= 96), -1 if t > 96
cudaError_t launch_pack_v_f16_only(const double* V, long long ldv, int t, int n, int n_pad, int npad, double scale,
                                   const void* vmax, double* colscale, void* vhi, void* vlo, cudaStream_t st);
cudaError_t launch_pack_v_f16(const double* V, long long ldv, int t, int n, int n_pad, int npad, double scale,
                              void* vmax, double* colscale, void* vhi, void* vlo, cudaStream_t st);
cudaError_t launch_fused_kmvm_tcg(int family, int d, int direct_dp, const float* xh, const float* xl,
                                  const float* xn, const float* x32, const void* vhi, const void* vlo,
                                  const double* colscale, double* out, const MvmArgs& a, int splits,
                                  cudaStream_t st);

// Reference-formula kernel column (kernels.hpp:235-243) / derivative column (:252-267), fp64.
// which < 0: K[:, p];  which == 0: outputscale;  1..d: lengthscale which-1.
// dense exact mLL pieces and the predictive mean's cross-kernel MVM (gpk_mvm.cu).
cudaError_t launch_dense_kernel(int family, const double* sx, const double* x, const double* sq, int n, int d,
                                int which, double o2, double fac, double* out, long long ldm, cudaStream_t st);
cudaError_t launch_sym_frob_partials(const double* A, long long lda, const double* B, long long ldb, int n,
                                     double* part, cudaStream_t st);
cudaError_t launch_cross_mvm(int family, const double* sa, const double* qa, int na, const double* sb,
                             const double* qb, int nb, int d, double o2, const double* v, double* out,
                             cudaStream_t st);
cudaError_t launch_kernel_column(int family, const double* sx, const double* x, const double* sq, int n, int d,
                                 long long p, int which, double o2, double fac, double* out, cudaStream_t st);

// Bilinear derivative contraction (backward pass, fast mode): for w = 0..d
//   quad[w] - cmix gamma[w] = sum_ab dK_w[a,b] (u_a u_b - cmix sum_i S[a,i] Z[b,i])
// (the gradient only needs this combination, cmix = n / l); returns the raw (unscaled) sums
// per CTA, dp + 1 of them; the host applies the factors.
// a-rows restricted to [a_begin, a_begin + a_rows) (this rank's shard), b over all n_pad rows.
cudaError_t launch_deriv_contract(bool fp64, int family, int dp, const void* X, const void* U, const void* Zt,
                                  int a_begin, int a_rows, int n_pad, int l, double cmix, double* partials,
                                  int* nblocks, cudaStream_t st);

}  // namespace gpk
