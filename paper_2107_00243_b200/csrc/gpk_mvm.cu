// Fused-MVM front end: operand packing, split-K reduction, shape selection,
// and the reference-formula kernel columns used by the pivoted Cholesky.
#include <cmath>

#include "gpk_linalg.h"
#include "gpk_mvm.cuh"
#include "gpk_ref_shape.cuh"

namespace gpk {

template <int FAM>
cudaError_t launch_fused_kmvm_fam(bool fp64, int dp, int mode, int tn, const void* X, const void* V, double* out,
                                  const MvmArgs& a, dim3 g, cudaStream_t st);

int dpad_for(int d) {
  if (d <= 4) return 4;
  if (d <= 12) return 12;
  if (d <= 20) return 20;
  if (d <= 32) return 32;
  return -1;
}

static int pick_tn(int need, const int* set, int nset) {
  for (int i = 0; i < nset; ++i)
    if (set[i] >= need) return set[i];
  return -1;
}

// Derivative launches use a coarser TN set (parity / reference-faithful path only).
MvmShape mvm_shape(int t, bool fp64, int mode) {
  static const int f32[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 16};
  static const int f32d[] = {1, 2, 4, 8, 16};
  static const int f64[] = {1, 2, 4, 8};
  const int need = (t + kNCG - 1) / kNCG;
  MvmShape s{};
  if (fp64) s.tn = pick_tn(need, f64, 4);
  else s.tn = mode == kModeValue ? pick_tn(need, f32, 12) : pick_tn(need, f32d, 5);
  if (s.tn < 0) return s;
  const int w = fp64 ? 2 : 4;
  const int tnp = (s.tn + w - 1) / w * w;
  s.cgs = (!fp64 && (tnp % 8) == 0) ? tnp + 4 : tnp;
  s.vld = kNCG * s.cgs;
  return s;
}

double prescale_c(int family) {
  const double l2e = 1.4426950408889634;
  switch (family) {
    case kRBF: return 0.5 * l2e;
    case kMatern12: return l2e * l2e;
    case kMatern32: return 3.0 * l2e * l2e;
    case kMatern52: return 5.0 * l2e * l2e;
  }
  return 1.0;
}

cudaError_t launch_fused_kmvm(bool fp64, int family, int dp, int mode, const void* X, const void* V, double* out,
                              const MvmArgs& a, int splits, cudaStream_t st) {
  const MvmShape sh = mvm_shape(a.t, fp64, mode);
  if (sh.tn < 0) return cudaErrorInvalidValue;
  dim3 g((a.row_end - a.row_begin + kBM - 1) / kBM, splits);
  switch (family) {
    case kRBF: return launch_fused_kmvm_fam<kRBF>(fp64, dp, mode, sh.tn, X, V, out, a, g, st);
    case kMatern12: return launch_fused_kmvm_fam<kMatern12>(fp64, dp, mode, sh.tn, X, V, out, a, g, st);
    case kMatern32: return launch_fused_kmvm_fam<kMatern32>(fp64, dp, mode, sh.tn, X, V, out, a, g, st);
    case kMatern52: return launch_fused_kmvm_fam<kMatern52>(fp64, dp, mode, sh.tn, X, V, out, a, g, st);
  }
  return cudaErrorInvalidValue;
}

// out[c][i] = sum_s part[s][c][i], fixed order s = 0..splits-1.
__global__ void reduce_splits_kernel(const double* __restrict__ part, int splits, long long sstride, int t, int n,
                                     long long ldp, double* __restrict__ out, long long ldo) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long total = static_cast<long long>(t) * n;
  if (idx >= total) return;
  const int c = static_cast<int>(idx / n);
  const int i = static_cast<int>(idx % n);
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += part[k * sstride + c * ldp + i];
  out[c * ldo + i] = s;
}

// Same sums, two rows per thread with 16-byte loads of the (L2-resident) partials: the
// partial leading dimension and split stride are even, so (c, 2i) is 16-byte aligned.
__global__ void reduce_splits2_kernel(const double* __restrict__ part, int splits, long long sstride, int t, int n,
                                      long long ldp, double* __restrict__ out, long long ldo) {
  const int n2 = (n + 1) >> 1;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(t) * n2) return;
  const int c = static_cast<int>(idx / n2);
  const int i = 2 * static_cast<int>(idx % n2);
  double s0 = 0.0, s1 = 0.0;
  const double* p = part + c * ldp + i;
#pragma unroll 4
  for (int k = 0; k < splits; ++k) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(p + k * sstride));
    s0 += v.x;
    s1 += v.y;
  }
  out[c * ldo + i] = s0;
  if (i + 1 < n) out[c * ldo + i + 1] = s1;
}

cudaError_t launch_reduce_splits(const double* part, int splits, long long sstride, int t, int n, long long ldpart,
                                 double* out, long long ldo, cudaStream_t st) {
  const int thr = 256;
  if ((ldpart & 1) == 0 && (sstride & 1) == 0 && (reinterpret_cast<uintptr_t>(part) & 15) == 0 && ldpart >= n + (n & 1)) {
    const long long total2 = static_cast<long long>(t) * ((n + 1) >> 1);
    reduce_splits2_kernel<<<static_cast<unsigned>((total2 + thr - 1) / thr), thr, 0, st>>>(part, splits, sstride, t,
                                                                                         n, ldpart, out, ldo);
    return cudaGetLastError();
  }
  const long long total = static_cast<long long>(t) * n;
  reduce_splits_kernel<<<static_cast<unsigned>((total + thr - 1) / thr), thr, 0, st>>>(part, splits, sstride, t, n,
                                                                                       ldpart, out, ldo);
  return cudaGetLastError();
}

// kernels.hpp:166-168: scaled_x = X / l, sqnorms = row squared norms; plus the
// packed row-major fp32 (pre-scaled) and fp64 operands of the fused MVM.
__global__ void pack_x_kernel(const double* __restrict__ X, long long ldx, int n, int d, int n_pad,
                              const double* __restrict__ ls, double prescale, int dp32, float* __restrict__ X32,
                              int dp64, double* __restrict__ X64s, double* __restrict__ sx, double* __restrict__ sq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  const double pre = sqrt(prescale);
  double acc = 0.0;
  for (int k = 0; k < dp32 || k < dp64; ++k) {
    double v = 0.0;
    if (i < n && k < d) {
      // the reference divides by the lengthscale (kernels.hpp:166)
      v = __ddiv_rn(X[k * ldx + i], ls[k]);
      sx[static_cast<long long>(k) * n + i] = v;
      acc = __dadd_rn(acc, __dmul_rn(v, v));
    }
    if (k < dp32) X32[static_cast<long long>(i) * dp32 + k] = static_cast<float>(v * pre);
    if (k < dp64) X64s[static_cast<long long>(i) * dp64 + k] = v;
  }
  if (i < n) sq[i] = acc;
}

cudaError_t launch_pack_x(const double* X, long long ldx, int n, int d, int n_pad, const double* ls,
                          double prescale, int dp32, float* X32, int dp64, double* X64s, double* sx, double* sq,
                          cudaStream_t st) {
  pack_x_kernel<<<(n_pad + 255) / 256, 256, 0, st>>>(X, ldx, n, d, n_pad, ls, prescale, dp32, X32, dp64, X64s, sx,
                                                      sq);
  return cudaGetLastError();
}

template <typename T>
__global__ void pack_v_kernel(const double* __restrict__ V, long long ldv, const int* __restrict__ colmap, int t,
                              int n, int n_pad, int tn, int cgs, int vld, T* __restrict__ out) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long total = static_cast<long long>(n_pad) * vld;
  if (idx >= total) return;
  const int i = static_cast<int>(idx / vld);
  const int e = static_cast<int>(idx % vld);
  const int g = e / cgs, q = e % cgs;
  const int c = g * tn + q;
  double v = 0.0;
  if (q < tn && c < t && i < n) {
    const int col = colmap ? colmap[c] : c;
    v = V[col * ldv + i];
  }
  out[idx] = static_cast<T>(v);
}

cudaError_t launch_pack_v32(const double* V, long long ldv, const int* colmap, int t, int n, int n_pad, MvmShape sh,
                            float* V32, cudaStream_t st) {
  const long long total = static_cast<long long>(n_pad) * sh.vld;
  pack_v_kernel<float><<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(V, ldv, colmap, t, n, n_pad, sh.tn,
                                                                                   sh.cgs, sh.vld, V32);
  return cudaGetLastError();
}

cudaError_t launch_pack_v64(const double* V, long long ldv, const int* colmap, int t, int n, int n_pad, MvmShape sh,
                            double* V64, cudaStream_t st) {
  const long long total = static_cast<long long>(n_pad) * sh.vld;
  pack_v_kernel<double><<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(V, ldv, colmap, t, n, n_pad,
                                                                                    sh.tn, sh.cgs, sh.vld, V64);
  return cudaGetLastError();
}

__global__ void kernel_column_kernel(int f, const double* __restrict__ sx, const double* __restrict__ x,
                                     const double* __restrict__ sq, int n, int d, long long p, int which, double o2,
                                     double fac, double* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double g = 0.0;
  for (int k = 0; k < d; ++k) g = __dadd_rn(g, __dmul_rn(sx[static_cast<long long>(k) * n + r], sx[k * n + p]));
  double s = __dsub_rn(__dadd_rn(sq[r], sq[p]), __dmul_rn(2.0, g));
  s = s > 0.0 ? s : 0.0;
  if (which < 0) {
    out[r] = __dmul_rn(o2, ref_shape(f, s));
  } else if (which == 0) {
    out[r] = __dmul_rn(fac, __dmul_rn(o2, ref_shape(f, s)));  // (2/o) * kernel_column
  } else {
    const int j = which - 1;
    const double dx = __dsub_rn(x[static_cast<long long>(j) * n + r], x[static_cast<long long>(j) * n + p]);
    out[r] = __dmul_rn(fac, __dmul_rn(ref_shape_ds(f, s), __dmul_rn(dx, dx)));
  }
}

cudaError_t launch_kernel_column(int family, const double* sx, const double* x, const double* sq, int n, int d,
                                 long long p, int which, double o2, double fac, double* out, cudaStream_t st) {
  kernel_column_kernel<<<(n + 255) / 256, 256, 0, st>>>(family, sx, x, sq, n, d, p, which, o2, fac, out);
  return cudaGetLastError();
}

// pivot column with the pivot index read from the device-resident state
__global__ void pchol_column_dev_kernel(int f, const double* __restrict__ sx, const double* __restrict__ sq, int n,
                                        int d, double o2, const PivotState* __restrict__ ps,
                                        double* __restrict__ out) {
  if (ps->stopped) return;
  const long long p = ps->p;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double g = 0.0;
  for (int k = 0; k < d; ++k) g = __dadd_rn(g, __dmul_rn(sx[static_cast<long long>(k) * n + r], sx[k * n + p]));
  double s = __dsub_rn(__dadd_rn(sq[r], sq[p]), __dmul_rn(2.0, g));
  s = s > 0.0 ? s : 0.0;
  out[r] = __dmul_rn(o2, ref_shape(f, s));
}

cudaError_t launch_pchol_column_dev(int f, const double* sx, const double* sq, int n, int d, double o2,
                                    const PivotState* ps, double* out, cudaStream_t st) {
  pchol_column_dev_kernel<<<(n + 63) / 64, 64, 0, st>>>(f, sx, sq, n, d, o2, ps, out);
  return cudaGetLastError();
}

// all derivative columns of pivot p at once: one thread per row evaluates the
// distance and both shape values once and writes the nw = d + 1 columns
__global__ void kernel_deriv_columns_kernel(int f, const double* __restrict__ sx, const double* __restrict__ x,
                                            const double* __restrict__ sq, int n, int d, long long p, int nw,
                                            const double* __restrict__ facs, double o2, double* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double g = 0.0;
  for (int k = 0; k < d; ++k) g = __dadd_rn(g, __dmul_rn(sx[static_cast<long long>(k) * n + r], sx[k * n + p]));
  double s = __dsub_rn(__dadd_rn(sq[r], sq[p]), __dmul_rn(2.0, g));
  s = s > 0.0 ? s : 0.0;
  out[r] = __dmul_rn(facs[0], __dmul_rn(o2, ref_shape(f, s)));
  if (nw > 1) {
    const double ds = ref_shape_ds(f, s);
    for (int w = 1; w < nw; ++w) {
      const int j = w - 1;
      const double dx = __dsub_rn(x[static_cast<long long>(j) * n + r], x[static_cast<long long>(j) * n + p]);
      out[static_cast<long long>(w) * n + r] = __dmul_rn(facs[w], __dmul_rn(ds, __dmul_rn(dx, dx)));
    }
  }
}

cudaError_t launch_kernel_deriv_columns(int family, const double* sx, const double* x, const double* sq, int n, int d,
                                        long long p, int nw, const double* facs, double o2, double* out,
                                        cudaStream_t st) {
  kernel_deriv_columns_kernel<<<(n + 127) / 128, 128, 0, st>>>(family, sx, x, sq, n, d, p, nw, facs, o2, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// dense exact mLL (validation / test metric, gp_likelihood.hpp:124-146)
// and the predictive mean's cross-kernel MVM (kernels.hpp:339-354, experiments.hpp:410-412).
// ---------------------------------------------------------------------------

// Dense noise-free K (which < 0) or dK/dtheta_which (0..d) in fp64, column-major
// [n][ldm]: entry (r, p) with the same operation order as kernel_column_kernel
// (the reference's assemble_kernel_rows / kernel_column expanded distances).
// Grid: x over rows (256 per block), y over columns.
__global__ void dense_kernel_kernel(int f, const double* __restrict__ sx, const double* __restrict__ x,
                                    const double* __restrict__ sq, int n, int d, int which, double o2, double fac,
                                    double* __restrict__ out, long long ldm) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const long long p = blockIdx.y;
  if (r >= n) return;
  double g = 0.0;
  for (int k = 0; k < d; ++k) g = __dadd_rn(g, __dmul_rn(sx[static_cast<long long>(k) * n + r], sx[k * n + p]));
  double s = __dsub_rn(__dadd_rn(sq[r], sq[p]), __dmul_rn(2.0, g));
  s = s > 0.0 ? s : 0.0;
  double v;
  if (which < 0) {
    v = __dmul_rn(o2, ref_shape(f, s));
  } else if (which == 0) {
    v = __dmul_rn(fac, __dmul_rn(o2, ref_shape(f, s)));
  } else {
    const int j = which - 1;
    const double dx = __dsub_rn(x[static_cast<long long>(j) * n + r], x[static_cast<long long>(j) * n + p]);
    v = __dmul_rn(fac, __dmul_rn(ref_shape_ds(f, s), __dmul_rn(dx, dx)));
  }
  out[p * ldm + r] = v;
}

cudaError_t launch_dense_kernel(int family, const double* sx, const double* x, const double* sq, int n, int d,
                                int which, double o2, double fac, double* out, long long ldm, cudaStream_t st) {
  dim3 g((n + 255) / 256, n);
  dense_kernel_kernel<<<g, 256, 0, st>>>(family, sx, x, sq, n, d, which, o2, fac, out, ldm);
  return cudaGetLastError();
}

// Per-block partial sums of sum_{i,j} A_ij B_ij for symmetric A, B of which only the
// LOWER triangles are valid (cuSOLVER potri / the assembled dK): diagonal once,
// strictly-lower entries twice.  One block per column j (fixed order: deterministic).
__global__ void sym_frob_partials_kernel(const double* __restrict__ A, long long lda, const double* __restrict__ B,
                                         long long ldb, int n, double* __restrict__ part) {
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int i = j + threadIdx.x; i < n; i += blockDim.x) {
    const double v = A[j * lda + i] * B[j * ldb + i];
    acc += (i == j) ? v : 2.0 * v;
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[j] = sh[0];
}

cudaError_t launch_sym_frob_partials(const double* A, long long lda, const double* B, long long ldb, int n,
                                     double* part, cudaStream_t st) {
  sym_frob_partials_kernel<<<n, 256, 0, st>>>(A, lda, B, ldb, n, part);
  return cudaGetLastError();
}

// out[i] = sum_j o2 shape(max(-2 <sa_i, sb_j> + |sa_i|^2 + |sb_j|^2, 0)) v[j]
// (cross_kernel(A, B) v, kernels.hpp:339-354) in fp64.  128 rows of A per block (one per
// thread, coordinates in registers), 64-row tiles of B and v staged in shared memory.
constexpr int kXR = 128, kXC = 64;
__global__ void __launch_bounds__(kXR) cross_mvm_kernel(int f, const double* __restrict__ sa,
                                                        const double* __restrict__ qa, int na,
                                                        const double* __restrict__ sb,
                                                        const double* __restrict__ qb, int nb, int d, double o2,
                                                        const double* __restrict__ v, double* __restrict__ out) {
  __shared__ double tb[32][kXC];
  __shared__ double tq[kXC], tv[kXC];
  const int i = blockIdx.x * kXR + threadIdx.x;
  double a[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) a[k] = (k < d && i < na) ? sa[static_cast<long long>(k) * na + i] : 0.0;
  const double qi = i < na ? qa[i] : 0.0;
  double acc = 0.0;
  for (int j0 = 0; j0 < nb; j0 += kXC) {
    __syncthreads();
    for (int e = threadIdx.x; e < d * kXC; e += kXR) {
      const int k = e / kXC, jj = e % kXC;
      tb[k][jj] = j0 + jj < nb ? sb[static_cast<long long>(k) * nb + j0 + jj] : 0.0;
    }
    if (threadIdx.x < kXC) {
      const int j = j0 + threadIdx.x;
      tq[threadIdx.x] = j < nb ? qb[j] : 0.0;
      tv[threadIdx.x] = j < nb ? v[j] : 0.0;
    }
    __syncthreads();
    const int jn = min(kXC, nb - j0);
    for (int jj = 0; jj < jn; ++jj) {
      double g = 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (k < d) g = __dadd_rn(g, __dmul_rn(a[k], tb[k][jj]));
      double s = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, g), qi), tq[jj]);
      s = s > 0.0 ? s : 0.0;
      acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(o2, ref_shape(f, s)), tv[jj]));
    }
  }
  if (i < na) out[i] = acc;
}

cudaError_t launch_cross_mvm(int family, const double* sa, const double* qa, int na, const double* sb,
                             const double* qb, int nb, int d, double o2, const double* v, double* out,
                             cudaStream_t st) {
  cross_mvm_kernel<<<(na + kXR - 1) / kXR, kXR, 0, st>>>(family, sa, qa, na, sb, qb, nb, d, o2, v, out);
  return cudaGetLastError();
}

}  // namespace gpk
