// Fused matrix-free kernel MVM:  out[:, c] = scale * sum_j k(x_i, x_j) V[j, c]
//
// Replaces KernelOperator::apply / deriv_apply (kernels.hpp:184-215) whose
// MatrixFree path assembles a 1024-row block of kernel entries in HBM-backed
// memory and runs one GEMV per column and per CG iteration.  Here every kernel
// entry is generated once per launch in registers/shared memory and contracted
// against all t right-hand-side columns of the mBCG block:
//
//   CTA = 256 threads, 128 output rows, all t columns, j-tiles of 32.
//   Per j-tile:  TMA bulk copies (cp.async.bulk + mbarrier, 3-stage ring) bring
//   X_j [32 x DP] and V_j [32 x VLD] into shared memory; phase 1: each thread
//   evaluates 16 kernel entries of its row (direct-difference distance,
//   MUFU ex2/sqrt) into a double-buffered K tile; phase 2: register-blocked
//   4 x TN outer products  acc[r][c] += K[r, j] * V[j, c].
//
// The per-(row, column) accumulation order depends only on n (never on t or
// on which other columns are present), so batched columns are bitwise equal
// to independent solves (the batched_pcg contract, krylov.hpp:131-132).
#pragma once
#include "gpk_common.cuh"
#include "gpk_internal.h"

namespace gpk {

constexpr int kBM = 128;  // output rows per CTA
constexpr int kBK = 32;   // j-tile
constexpr int kNCG = 8;   // column groups per CTA
constexpr int kStages = 3;
constexpr int kThreads = 256;

template <typename T>
struct VecT;
template <>
struct VecT<float> {
  using V = float4;
  static constexpr int W = 4;
};
template <>
struct VecT<double> {
  using V = double2;
  static constexpr int W = 2;
};

// Column-group stride (elements) of the packed V layout; padded to dodge
// shared-memory bank conflicts between the 8 column groups of a warp.
template <typename T, int TN>
struct VLayout {
  static constexpr int W = VecT<T>::W;
  static constexpr int TNP = (TN + W - 1) / W * W;
  static constexpr int CGS = (sizeof(T) == 4 && (TNP % 8) == 0) ? TNP + 4 : TNP;
  static constexpr int VLD = kNCG * CGS;
};

// ---- kernel shape functions -------------------------------------------------
// FP32: coordinates are pre-scaled by sqrt(c_fam) so s' = c_fam * s (see
// prescale_factor) and exp becomes a single MUFU.EX2.
template <int FAM>
GPK_DEV float kval32(float s) {
  if constexpr (FAM == kRBF) {
    return ex2_approx(-s);
  } else {
    const float r = sqrt_approx(s);
    const float e = ex2_approx(-r);
    if constexpr (FAM == kMatern12) return e;
    if constexpr (FAM == kMatern32) return fmaf(r, kLn2, 1.0f) * e;
    const float rr = r * kLn2;  // Matern52
    return fmaf(rr, fmaf(rr, 1.0f / 3.0f, 1.0f), 1.0f) * e;
  }
}
// C * kval32(s) with the constant folded into the shape polynomial (RBF: into the
// ex2 argument when C is a power of two, passed as log2 C).
template <int FAM, int LOG2C>
GPK_DEV float kval32_scaled(float s) {
  constexpr float C = static_cast<float>(1 << LOG2C);
  if constexpr (FAM == kRBF) {
    return ex2_approx(static_cast<float>(LOG2C) - s);
  } else {
    const float r = sqrt_approx(s);
    const float e = ex2_approx(-r);
    if constexpr (FAM == kMatern12) return C * e;
    if constexpr (FAM == kMatern32) return fmaf(r, C * kLn2, C) * e;
    const float rr = r * kLn2;  // Matern52
    return fmaf(rr, fmaf(rr, C / 3.0f, C), C) * e;
  }
}
// kval32_scaled for two entries at once: the FP32 polynomial / scaling steps as paired
// FFMA2 / FMUL2 (one instruction per two entries), the sqrt / ex2 on the SFU per entry.
template <int FAM, int LOG2C>
GPK_DEV float2 kval32x2_scaled(float2 s) {
  constexpr float C = static_cast<float>(1 << LOG2C);
  if constexpr (FAM == kRBF) {
    const float2 a = __fadd2_rn(make_float2(static_cast<float>(LOG2C), static_cast<float>(LOG2C)),
                                make_float2(-s.x, -s.y));
    return make_float2(ex2_approx(a.x), ex2_approx(a.y));
  } else {
    const float2 r = make_float2(sqrt_approx(s.x), sqrt_approx(s.y));
    const float2 e = make_float2(ex2_approx(-r.x), ex2_approx(-r.y));
    if constexpr (FAM == kMatern12) return __fmul2_rn(make_float2(C, C), e);
    if constexpr (FAM == kMatern32)
      return __fmul2_rn(__ffma2_rn(r, make_float2(C * kLn2, C * kLn2), make_float2(C, C)), e);
    const float2 rr = __fmul2_rn(r, make_float2(kLn2, kLn2));  // Matern52
    const float2 q = __ffma2_rn(rr, make_float2(C / 3.0f, C / 3.0f), make_float2(C, C));
    return __fmul2_rn(__ffma2_rn(rr, q, make_float2(C, C)), e);
  }
}
// shape_ds (kernels.hpp:115-134) in pre-scaled units.
template <int FAM>
GPK_DEV float kds32(float s) {
  if constexpr (FAM == kRBF) {
    return -0.5f * ex2_approx(-s);
  } else {
    const float r = sqrt_approx(s);
    const float e = ex2_approx(-r);
    if constexpr (FAM == kMatern12) return s > 0.0f ? -e * kLog2e / (2.0f * r) : 0.0f;
    if constexpr (FAM == kMatern32) return -1.5f * e;
    return -(5.0f / 6.0f) * fmaf(r, kLn2, 1.0f) * e;  // Matern52
  }
}
// FP64: the reference's own shape / shape_ds on unscaled s (kernels.hpp:93-134).
template <int FAM>
GPK_DEV double kval64(double s) {
  if constexpr (FAM == kRBF) return exp(-0.5 * s);
  if constexpr (FAM == kMatern12) return exp(-sqrt(s));
  if constexpr (FAM == kMatern32) {
    const double r = sqrt(3.0 * s);
    return (1.0 + r) * exp(-r);
  }
  const double r = sqrt(5.0 * s);
  return (1.0 + r + r * r / 3.0) * exp(-r);
}
template <int FAM>
GPK_DEV double kds64(double s) {
  if constexpr (FAM == kRBF) return -0.5 * exp(-0.5 * s);
  if constexpr (FAM == kMatern12) {
    if (s <= 0.0) return 0.0;
    const double r = sqrt(s);
    return -exp(-r) / (2.0 * r);
  }
  if constexpr (FAM == kMatern32) return -1.5 * exp(-sqrt(3.0 * s));
  const double r = sqrt(5.0 * s);
  return -(5.0 / 6.0) * (1.0 + r) * exp(-r);
}

template <typename T, int FAM, int MODE>
GPK_DEV T kentry(T s, T dsel) {
  if constexpr (sizeof(T) == 4) {
    if constexpr (MODE == kModeValue) return kval32<FAM>(s);
    else return kds32<FAM>(s) * (dsel * dsel);
  } else {
    if constexpr (MODE == kModeValue) return kval64<FAM>(s);
    else return kds64<FAM>(s) * (dsel * dsel);
  }
}

// ---------------------------------------------------------------------------
template <typename T, int FAM, int DP, int TN, int MODE>
// 2 CTAs (16 warps) per SM: <= 128 registers per thread
__global__ void __launch_bounds__(kThreads, (sizeof(T) == 4 && TN <= 9) ? 2 : 1)
    fused_kmvm_kernel(const T* __restrict__ X, const T* __restrict__ V, double* __restrict__ out, MvmArgs a) {
  using L = VLayout<T, TN>;
  using Vec = typename VecT<T>::V;
  constexpr int W = VecT<T>::W;
  constexpr int VLD = L::VLD;
  constexpr uint32_t kXBytes = kBK * DP * sizeof(T);
  constexpr uint32_t kVBytes = kBK * VLD * sizeof(T);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  T* Xs = reinterpret_cast<T*>(smem_raw + 128);
  T* Vs = Xs + kStages * kBK * DP;
  T* Ks = Vs + kStages * kBK * VLD;

  const int tid = threadIdx.x;
  const int row0 = a.row_begin + blockIdx.x * kBM;
  const int jt0 = blockIdx.y * a.jtiles_per_split;
  const int jt1 = min(jt0 + a.jtiles_per_split, a.n_pad / kBK);
  const int nt = jt1 - jt0;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int stage, int jt) {
    const long long j0 = static_cast<long long>(jt) * kBK;
    mbar_arrive_expect_tx(&bar[stage], kXBytes + kVBytes);
    bulk_g2s(Xs + stage * kBK * DP, X + j0 * DP, kXBytes, &bar[stage]);
    bulk_g2s(Vs + stage * kBK * VLD, V + j0 * VLD, kVBytes, &bar[stage]);
  };
  if (tid == 0)
    for (int s = 0; s < kStages && s < nt; ++s) issue(s, jt0 + s);

  // phase-1 role: one row, half of the j-tile
  const int pr = tid & (kBM - 1);
  const int ph = tid >> 7;
  T xr[DP];
  {
    const Vec* src = reinterpret_cast<const Vec*>(X + static_cast<long long>(row0 + pr) * DP);
#pragma unroll
    for (int k = 0; k < DP / W; ++k) {
      const Vec v = src[k];
      if constexpr (W == 4) {
        xr[4 * k] = v.x; xr[4 * k + 1] = v.y; xr[4 * k + 2] = v.z; xr[4 * k + 3] = v.w;
      } else {
        xr[2 * k] = v.x; xr[2 * k + 1] = v.y;
      }
    }
  }
  // phase-2 role: 4 rows x TN columns
  const int cg = tid & (kNCG - 1);
  const int rg = tid >> 3;
  T acc[4][TN];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[r][c] = T(0);
  double acc64[sizeof(T) == 4 ? 4 : 1][sizeof(T) == 4 ? TN : 1];
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < TN; ++c) acc64[r][c] = 0.0;
  }

  // one kernel entry K[pr, j] of the tile staged in xs (two partial sums
  // shorten the FFMA dependency chain of the distance)
  auto entry_at = [&](const T* xs, int j) -> T {
    const Vec* xj = reinterpret_cast<const Vec*>(xs + j * DP);
    T s0 = T(0), s1 = T(0), dsel = T(0);
#pragma unroll
    for (int k = 0; k < DP / W; ++k) {
      const Vec v = xj[k];
      T df[W];
      if constexpr (W == 4) {
        df[0] = xr[4 * k] - v.x; df[1] = xr[4 * k + 1] - v.y; df[2] = xr[4 * k + 2] - v.z; df[3] = xr[4 * k + 3] - v.w;
      } else {
        df[0] = xr[2 * k] - v.x; df[1] = xr[2 * k + 1] - v.y;
      }
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (q & 1) s1 = fma(df[q], df[q], s1);
        else s0 = fma(df[q], df[q], s0);
        if constexpr (MODE == kModeDls) dsel = (W * k + q == a.jdim) ? df[q] : dsel;
      }
    }
    return kentry<T, FAM, MODE>(s0 + s1, dsel);
  };
  // one rank-1 update of the 4 x TN register tile
  auto mma_step = [&](const T* kb, const T* vs, int kk) {
    T av[4];
    if constexpr (W == 4) {
      const float4 t4 = *reinterpret_cast<const float4*>(kb + kk * kBM + rg * 4);
      av[0] = t4.x; av[1] = t4.y; av[2] = t4.z; av[3] = t4.w;
    } else {
      const double2 t0 = *reinterpret_cast<const double2*>(kb + kk * kBM + rg * 4);
      const double2 t1 = *reinterpret_cast<const double2*>(kb + kk * kBM + rg * 4 + 2);
      av[0] = t0.x; av[1] = t0.y; av[2] = t1.x; av[3] = t1.y;
    }
    T bv[L::TNP];
    const Vec* vrow = reinterpret_cast<const Vec*>(vs + kk * VLD);
#pragma unroll
    for (int q = 0; q < L::TNP / W; ++q) {
      const Vec v = vrow[q];
      if constexpr (W == 4) {
        bv[4 * q] = v.x; bv[4 * q + 1] = v.y; bv[4 * q + 2] = v.z; bv[4 * q + 3] = v.w;
      } else {
        bv[2 * q] = v.x; bv[2 * q + 1] = v.y;
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < TN; ++c) acc[r][c] = fma(av[r], bv[c], acc[r][c]);
  };

  // prologue: entries of tile 0
  if (nt > 0) {
    mbar_wait(&bar[0], 0);
#pragma unroll 2
    for (int q = 0; q < kBK / 2; ++q) {
      const int j = ph * (kBK / 2) + q;
      Ks[j * kBM + pr] = entry_at(Xs, j);
    }
  }
  __syncthreads();

  // steady state: contraction of tile `it` software-pipelined with the entries of tile it+1
  for (int it = 0; it < nt; ++it) {
    const int stage = it % kStages;
    const bool has_next = it + 1 < nt;
    const int nstage = (it + 1) % kStages;
    if (has_next) mbar_wait(&bar[nstage], ((it + 1) / kStages) & 1);
    const T* kb = Ks + (it & 1) * (kBK * kBM);
    T* kn = Ks + ((it + 1) & 1) * (kBK * kBM);
    const T* xsn = Xs + nstage * kBK * DP;
    const T* vs = Vs + stage * kBK * VLD + cg * L::CGS;
    if (has_next) {
#pragma unroll 2
      for (int q = 0; q < kBK / 2; ++q) {
        const int j = ph * (kBK / 2) + q;
        kn[j * kBM + pr] = entry_at(xsn, j);
        mma_step(kb, vs, 2 * q);
        mma_step(kb, vs, 2 * q + 1);
      }
    } else {
#pragma unroll 4
      for (int kk = 0; kk < kBK; ++kk) mma_step(kb, vs, kk);
    }
    if constexpr (sizeof(T) == 4) {
      // fp32 within 4 j-tiles (128 entries), fp64 across them
      if ((it & 3) == 3 || it == nt - 1) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < TN; ++c) {
            acc64[r][c] += static_cast<double>(acc[r][c]);
            acc[r][c] = 0.0f;
          }
      }
    }
    __syncthreads();  // tile `it` fully consumed (X in the previous iteration, V now); K[it+1] complete
    if (tid == 0 && it + kStages < nt) {
      fence_proxy_async();
      issue(stage, jt0 + it + kStages);
    }
  }

  // ---- epilogue: column-major fp64 output (or split-K partial)
  double* o = out + static_cast<long long>(blockIdx.y) * a.split_stride;
#pragma unroll
  for (int c = 0; c < TN; ++c) {
    const int col = cg * TN + c;
    if (col >= a.t) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = row0 + rg * 4 + r;
      if (row < a.row_end) {
        double v;
        if constexpr (sizeof(T) == 4) v = acc64[r][c];
        else v = static_cast<double>(acc[r][c]);
        o[static_cast<long long>(col) * a.ldo + (row - a.row_begin)] = a.scale * v;
      }
    }
  }
}

template <typename T, int FAM, int DP, int TN, int MODE>
size_t fused_kmvm_smem() {
  using L = VLayout<T, TN>;
  return 128 + sizeof(T) * (kStages * kBK * DP + kStages * kBK * L::VLD + 2 * kBK * kBM);
}

template <typename T, int FAM, int DP, int TN, int MODE>
cudaError_t launch_fused_kmvm_t(const T* X, const T* V, double* out, const MvmArgs& a, dim3 grid,
                                cudaStream_t st) {
  const size_t sm = fused_kmvm_smem<T, FAM, DP, TN, MODE>();
  auto k = fused_kmvm_kernel<T, FAM, DP, TN, MODE>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k<<<grid, kThreads, sm, st>>>(X, V, out, a);
  return cudaGetLastError();
}

}  // namespace gpk
