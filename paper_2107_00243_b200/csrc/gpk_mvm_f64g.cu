// FP64 kernel MVM on the fp64 tensor cores (DMMA 8x8x4), value mode:
//   out[i, c] = sum_j o^2 shape(s_ij) V[j, c],   s_ij = max(0, (-2 <xs_i, xs_j> + |xs_i|^2) + |xs_j|^2)
// i.e. KernelOperator::apply's MatrixFree block (kernels.hpp:296-306) with the reference's own
// expanded distance and shape operation order (ref_shape, kernels.hpp:93-111).  It is the
// fp64 parity operator and the fp64 residual of the certified defect correction.
//
// Structure (one warp = 8 output rows x up to 64 columns, CTA = 8 warps = 64 rows):
//   per 8-wide j sub-tile: Gram tile G = X_i X_j^T with dp/4 DMMAs (A fragments of the warp's
//   rows held in registers, B fragments from the shared-memory X_j tile), then each lane turns
//   its two accumulator values D[m][2r], D[m][2r+1] into kernel entries and uses them directly
//   as the A fragments of two contraction k-steps (K index order {0,2,4,6}, {1,3,5,7}); near
//   pairs (s <= (|x_i|^2 + |x_j|^2) / 16) redo the inner product sequentially, as the
//   reference does, from the staged rows.  The matching V fragments are one 128-bit shared load (V staged as [column][j]).  No kernel
//   tile ever leaves registers.  X_j, |x_j|^2 and V_j chunks of 64 rows are double-buffered
//   with cp.async.  Each output is a fixed-order sum over j (chunk, sub-tile, DMMA) that
//   depends on n only: batched columns are bitwise equal to independent ones
//   (krylov.hpp:131-132), and row shards reproduce the unsharded rows bitwise.
// The earlier fp64 operator (fused_kmvm_kernel<double>, direct differences on the FP64 FMA
// pipe) took 5.3 ms at C2 (n = 16384, d = 18, t = 51).
#include <algorithm>
#include <cstdint>

#include "gpk_common.cuh"
#include "gpk_internal.h"
#include "gpk_ref_shape.cuh"

namespace gpk {

namespace {

constexpr int kFT = 256;  // threads (8 warps)
constexpr int kFJ = 64;   // j rows per staged chunk
constexpr int kFV = 72;   // V tile stride (doubles): 36 = 4 (mod 8) 16-byte units -> conflict-free LDS.128

GPK_DEV void dmma_f(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <bool VEC>
GPK_DEV void cp_pair_f(double* dst, const double* src, int nv, const double* safe) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if (VEC) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(nv > 0 ? src : safe),
                 "r"(nv >= 2 ? 16 : nv * 8)
                 : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(nv > 0 ? src : safe),
                 "r"(nv > 0 ? 8 : 0)
                 : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d + 8), "l"(nv > 1 ? src + 1 : safe),
                 "r"(nv > 1 ? 8 : 0)
                 : "memory");
  }
}
GPK_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
GPK_DEV void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
GPK_DEV void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// X_j row stride in shared memory: = 4 (mod 16) doubles, so the Gram B fragments are
// conflict-free 64-bit loads
constexpr int xstride(int dp) { return (dp - 4 + 15) / 16 * 16 + 4; }

}  // namespace

template <int FAM, int DP, int NT, bool VEC>
__global__ void __launch_bounds__(kFT, 2)
    fused_kmvm_f64g_kernel(const double* __restrict__ X, const double* __restrict__ sq, int n,
                           const double* __restrict__ V, long long ldv, int tc, double* __restrict__ out,
                           long long ldo, double scale, int row_begin, int row_end) {
  constexpr int XS = xstride(DP);
  constexpr int KQ = DP / 4;
  extern __shared__ __align__(16) double fsm[];
  double* Xs = fsm;                      // [2][kFJ][XS]
  double* Ss = Xs + 2 * kFJ * XS;        // [2][kFJ]
  double* Vs = Ss + 2 * kFJ;             // [2][NT * 8][kFV]
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, r = lane & 3, m = lane >> 2;
  const int i0 = row_begin + blockIdx.x * 64 + w * 8;
  const int row = i0 + m;
  // A fragments of the warp's rows (zero rows beyond row_end are harmless: not stored)
  double xa[KQ];
#pragma unroll
  for (int q = 0; q < KQ; ++q) xa[q] = row < n ? X[static_cast<long long>(row) * DP + 4 * q + r] : 0.0;
  const double sqi = row < n ? sq[row] : 0.0;
  double acc[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;

  const int nchunks = (n + kFJ - 1) / kFJ;
  auto stage = [&](int buf, int ch) {
    const int j0 = ch * kFJ;
    double* xs = Xs + buf * kFJ * XS;
    // X_j: kFJ rows x DP doubles, contiguous in global memory (padded rows beyond n are zero)
    for (int e = tid; e < kFJ * DP / 2; e += kFT) {
      const int jr = e / (DP / 2), kp = e % (DP / 2);
      const int j = j0 + jr;
      cp_pair_f<true>(xs + jr * XS + 2 * kp, X + static_cast<long long>(min(j, n - 1)) * DP + 2 * kp, j < n ? 2 : 0,
                      X);
    }
    if (tid < kFJ / 2) {
      const int j = j0 + 2 * tid;
      cp_pair_f<false>(Ss + buf * kFJ + 2 * tid, sq + min(j, n - 1), min(2, max(0, n - j)), sq);
    }
    // V_j: column c, rows j0 .. j0 + 63 (zero beyond n; columns >= tc duplicate the last)
    double* vs = Vs + buf * NT * 8 * kFV;
    for (int e = tid; e < NT * 8 * (kFJ / 2); e += kFT) {
      const int c = e / (kFJ / 2), jp = e % (kFJ / 2);
      const int j = j0 + 2 * jp;
      cp_pair_f<VEC>(vs + c * kFV + 2 * jp, V + static_cast<long long>(min(c, tc - 1)) * ldv + min(j, n - 1),
                     min(2, max(0, n - j)), V);
    }
  };
  stage(0, 0);
  cp_commit();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) stage(buf ^ 1, ch + 1);
    cp_commit();
    cp_wait1();
    __syncthreads();
    const double* xs = Xs + buf * kFJ * XS;
    const double* ss = Ss + buf * kFJ;
    const double* vs = Vs + buf * NT * 8 * kFV;
#pragma unroll 2
    for (int jj = 0; jj < kFJ / 8; ++jj) {
      double g[2] = {0.0, 0.0};
#pragma unroll
      for (int q = 0; q < KQ; ++q) dmma_f(g, xa[q], xs[(jj * 8 + m) * XS + 4 * q + r]);
      const double2 sj = *reinterpret_cast<const double2*>(ss + jj * 8 + 2 * r);
      double kv[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {  // kernels.hpp:298-301: ((-2 g) + |x_i|^2) + |x_j|^2, clamped
        const double sqj = e ? sj.y : sj.x;
        double s = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, g[e]), sqi), sqj);
        if (s <= 0.0625 * (sqi + sqj)) {
          // near pair (the diagonal included): the cancellation amplifies the DMMA's own
          // rounding, so the inner product is redone in the reference's sequential order
          // (kernels.hpp:298, bitwise equal to |x|^2 on the diagonal -> s = 0 exactly)
          const double* xi = X + static_cast<long long>(row < n ? row : 0) * DP;
          const double* xj = xs + (jj * 8 + 2 * r + e) * XS;
          double gs = 0.0;
#pragma unroll
          for (int k = 0; k < DP; ++k) gs = __dadd_rn(gs, __dmul_rn(xi[k], xj[k]));
          s = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, gs), sqi), sqj);
        }
        s = s > 0.0 ? s : 0.0;
        kv[e] = __dmul_rn(scale, ref_shape(FAM, s));
      }
      double2 b[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = *reinterpret_cast<const double2*>(vs + (nt * 8 + m) * kFV + jj * 8 + 2 * r);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma_f(acc[nt], kv[0], b[nt].x);  // independent accumulators first
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma_f(acc[nt], kv[1], b[nt].y);
    }
    __syncthreads();  // buffer buf is refilled at the next iteration
  }
  cp_wait0();
  if (row < row_end) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = nt * 8 + 2 * r + e;
        if (c < tc) out[static_cast<long long>(c) * ldo + (row - row_begin)] = acc[nt][e];
      }
  }
}

namespace {

template <int FAM, int DP, int NT, bool VEC>
cudaError_t f64g_launch(const double* X, const double* sq, int n, const double* V, long long ldv, int tc,
                        double* out, long long ldo, double scale, int row_begin, int row_end, cudaStream_t st) {
  constexpr int XS = xstride(DP);
  const size_t smem = sizeof(double) * (2 * kFJ * XS + 2 * kFJ + 2 * NT * 8 * kFV);
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = cudaFuncSetAttribute(fused_kmvm_f64g_kernel<FAM, DP, NT, VEC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const int rows = row_end - row_begin;
  fused_kmvm_f64g_kernel<FAM, DP, NT, VEC><<<(rows + 63) / 64, kFT, smem, st>>>(X, sq, n, V, ldv, tc, out, ldo, scale,
                                                                               row_begin, row_end);
  return cudaGetLastError();
}

template <int FAM, int DP, bool VEC>
cudaError_t f64g_nt(int nt, const double* X, const double* sq, int n, const double* V, long long ldv, int tc,
                    double* out, long long ldo, double scale, int row_begin, int row_end, cudaStream_t st) {
#define GPK_F64G(NTV) \
  case NTV:           \
    return f64g_launch<FAM, DP, NTV, VEC>(X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
  switch (nt) {
    GPK_F64G(1) GPK_F64G(2) GPK_F64G(3) GPK_F64G(4) GPK_F64G(5) GPK_F64G(6) GPK_F64G(7) GPK_F64G(8) GPK_F64G(9)
  }
#undef GPK_F64G
  return cudaErrorInvalidValue;
}

template <int FAM, bool VEC>
cudaError_t f64g_dp(int dp, int nt, const double* X, const double* sq, int n, const double* V, long long ldv, int tc,
                    double* out, long long ldo, double scale, int row_begin, int row_end, cudaStream_t st) {
  switch (dp) {
    case 4: return f64g_nt<FAM, 4, VEC>(nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
    case 12: return f64g_nt<FAM, 12, VEC>(nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
    case 20: return f64g_nt<FAM, 20, VEC>(nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
    case 32: return f64g_nt<FAM, 32, VEC>(nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
  }
  return cudaErrorInvalidValue;
}

template <bool VEC>
cudaError_t f64g_fam(int family, int dp, int nt, const double* X, const double* sq, int n, const double* V,
                     long long ldv, int tc, double* out, long long ldo, double scale, int row_begin, int row_end,
                     cudaStream_t st) {
  switch (family) {
    case kRBF: return f64g_dp<kRBF, VEC>(dp, nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
    case kMatern12:
      return f64g_dp<kMatern12, VEC>(dp, nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
    case kMatern32:
      return f64g_dp<kMatern32, VEC>(dp, nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
    case kMatern52:
      return f64g_dp<kMatern52, VEC>(dp, nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// X: packed fp64 scaled rows [n_pad][dp] (zero padding), sq: reference squared norms (n),
// V: column-major [tc][ldv] with all n rows, tc <= 72 (t = l + 1 = 65 at C5 in one launch: the
// entry evaluation, not the column count, sets the cost); out rows [row_begin, row_end).
cudaError_t launch_fused_kmvm_f64g(int family, int dp, const double* X, const double* sq, int n, const double* V,
                                   long long ldv, int tc, double* out, long long ldo, double scale, int row_begin,
                                   int row_end, cudaStream_t st) {
  if (tc <= 0 || row_end <= row_begin) return cudaSuccess;
  if (tc > 72) return cudaErrorInvalidValue;
  const int nt = (tc + 7) / 8;
  const bool vec = (reinterpret_cast<uintptr_t>(V) & 15) == 0 && ldv % 2 == 0;
  return vec ? f64g_fam<true>(family, dp, nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st)
             : f64g_fam<false>(family, dp, nt, X, sq, n, V, ldv, tc, out, ldo, scale, row_begin, row_end, st);
}

}  // namespace gpk
