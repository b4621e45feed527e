// Fused derivative pass (backward, bilinear form).
//
// The reference's backward pass (gp_likelihood.hpp:87-101 ->
// trace_estimation.hpp:190-224) runs one PCG solve K_hat w = dK_w z_i per
// hyperparameter and probe ((d+1) l solves) and one deriv_apply per parameter
// for u' dK_w u.  Because K_hat^{-1} is symmetric,
//     z_i' K_hat^{-1} dK_w z_i = s_i' dK_w z_i   with s_i = K_hat^{-1} z_i,
// the forward probe solutions (which the reference already keeps,
// trace_estimation.hpp:171) give every stochastic term in ONE pass over the
// n^2 kernel entries:
//     quad[w]  = sum_ab dK_w[a,b] u_a u_b
//     gamma[w] = sum_ab dK_w[a,b] W_ab,   W_ab = sum_i S[a,i] Z[b,i]
// with dK_0 = 2 o shape(s) and dK_{l_j} = (-2 o^2 / l_j) shape_ds(s) ds_j^2.  The gradient
// (gp_likelihood.hpp:97-100) needs them only as quad[w] - (n/l) gamma[w], so every pair
// contributes the single weight u_a u_b - (n/l) W_ab: one accumulator per hyperparameter.
//
// CTA = 256 threads = 16 x 16 threads, each owning a 4 x 4 tile of (a, b)
// pairs of a 64 x 64 block tile; W tiles come from register-blocked outer
// products over the l probe columns staged in shared memory; per-thread fp32
// sums of one b-tile are flushed into fp64 accumulators.
#include "gpk_common.cuh"
#include "gpk_internal.h"

namespace gpk {

constexpr int kDA = 64;  // a rows per block tile
constexpr int kDB = 64;  // b cols per block tile
constexpr int kDThreads = 256;
constexpr int kDBTilesPerBlock = 16;  // b-tiles handled by one CTA (fixed -> deterministic)

template <typename T, int FAM>
GPK_DEV void shape_pair(T s, T& e, T& ds) {
  if constexpr (sizeof(T) == 4) {
    if constexpr (FAM == kRBF) {
      e = ex2_approx(-s);
      ds = -0.5f * e;
    } else {
      const float r = sqrt_approx(s);
      const float x = ex2_approx(-r);
      if constexpr (FAM == kMatern12) {
        e = x;
        ds = s > 0.0f ? -x * kLog2e / (2.0f * r) : 0.0f;
      } else if constexpr (FAM == kMatern32) {
        e = fmaf(r, kLn2, 1.0f) * x;
        ds = -1.5f * x;
      } else {
        const float rr = r * kLn2;
        e = fmaf(rr, fmaf(rr, 1.0f / 3.0f, 1.0f), 1.0f) * x;
        ds = -(5.0f / 6.0f) * (1.0f + rr) * x;
      }
    }
  } else {
    if constexpr (FAM == kRBF) {
      e = exp(-0.5 * s);
      ds = -0.5 * e;
    } else if constexpr (FAM == kMatern12) {
      const double r = sqrt(s);
      e = exp(-r);
      ds = s > 0.0 ? -e / (2.0 * r) : 0.0;
    } else if constexpr (FAM == kMatern32) {
      const double r = sqrt(3.0 * s);
      const double x = exp(-r);
      e = (1.0 + r) * x;
      ds = -1.5 * x;
    } else {
      const double r = sqrt(5.0 * s);
      const double x = exp(-r);
      e = (1.0 + r + r * r / 3.0) * x;
      ds = -(5.0 / 6.0) * (1.0 + r) * x;
    }
  }
}

// X: [n_pad][DP] packed scaled coordinates (fp32 pre-scaled / fp64 plain);
// U: [n_pad]; S, Z: column-major [l][n_pad] (zero in padded rows).
// partials: per CTA, DP+1 doubles = {M0, M_1..M_DP}, M = Q - cmix G.
template <typename T, int FAM, int DP>
__global__ void __launch_bounds__(kDThreads, 1)
    deriv_contract_kernel(const T* __restrict__ X, const T* __restrict__ U, const T* __restrict__ S,
                          const T* __restrict__ Z, int n_pad, int l, int a_begin, T cmix,
                          double* __restrict__ partials) {
  constexpr int NA = DP + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Ss = reinterpret_cast<T*>(smem_raw);  // [l][kDA]
  T* Xa = Ss + l * kDA;                    // [kDA][DP]
  T* Ua = Xa + kDA * DP;                   // [kDA]
  T* Bbuf = Ua + kDA;                      // 2 x {Zs [l][kDB], Xb [kDB][DP], Ub [kDB]}: double-buffered b-tiles
  const int bstride = l * kDB + kDB * DP + kDB;
  __shared__ double red[kDThreads / 32];

  const int tid = threadIdx.x;
  const int ta = tid & 15;  // a-group (4 rows)
  const int tb = tid >> 4;  // b-group (4 cols)
  const int a0 = a_begin + blockIdx.x * kDA;  // this rank's a-rows (tiles never straddle shards)
  const int nbt = n_pad / kDB;
  const int bt0 = blockIdx.y * kDBTilesPerBlock;
  const int bt1 = min(bt0 + kDBTilesPerBlock, nbt);

  // b-tile staging with 16-byte cp.async (every row segment is 16-byte aligned: n_pad % 128 == 0)
  constexpr int V = 16 / sizeof(T);  // elements per copy
  auto cp16 = [](T* dst, const T* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  };
  auto stage = [&](int buf, int bt) {
    const int b0 = bt * kDB;
    T* zs = Bbuf + buf * bstride;
    T* xb = zs + l * kDB;
    T* ub = xb + kDB * DP;
    for (int e = tid; e < l * (kDB / V); e += kDThreads) {
      const int i = e / (kDB / V), r = (e % (kDB / V)) * V;
      cp16(zs + i * kDB + r, Z + static_cast<long long>(i) * n_pad + b0 + r);
    }
    for (int e = tid; e < kDB * DP / V; e += kDThreads) cp16(xb + e * V, X + static_cast<long long>(b0) * DP + e * V);
    for (int e = tid; e < kDB / V; e += kDThreads) cp16(ub + e * V, U + b0 + e * V);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (bt0 < bt1) stage(0, bt0);

  // a-tile operands (once per CTA)
  for (int e = tid; e < l * kDA; e += kDThreads) {
    const int i = e / kDA, r = e % kDA;
    Ss[e] = S[static_cast<long long>(i) * n_pad + a0 + r];
  }
  for (int e = tid; e < kDA * DP; e += kDThreads) Xa[e] = X[static_cast<long long>(a0) * DP + e];
  for (int e = tid; e < kDA; e += kDThreads) Ua[e] = U[a0 + e];

  double acc64[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) acc64[q] = 0.0;

  for (int bt = bt0; bt < bt1; ++bt) {
    const int buf = (bt - bt0) & 1;
    if (bt + 1 < bt1) {
      stage(buf ^ 1, bt + 1);  // the other buffer was released by the previous iteration's barrier
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // tile bt visible to every thread
    const T* Zs = Bbuf + buf * bstride;
    const T* Xb = Zs + l * kDB;
    const T* Ub = Xb + kDB * DP;

    // W tile (4 x 4 per thread) = S[a, :] . Z[b, :]
    T w[4][4];
    if constexpr (sizeof(T) == 4) {
      // fp32: paired FFMA2 (two b columns per instruction): half the issue slots of the rank-l product
      float2 w2[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r) w2[r][0] = w2[r][1] = make_float2(0.0f, 0.0f);
#pragma unroll 5
      for (int i = 0; i < l; ++i) {  // unrolled: the shared loads of later i are in flight early
        const float4 va = *reinterpret_cast<const float4*>(Ss + i * kDA + ta * 4);
        const float4 vb = *reinterpret_cast<const float4*>(Zs + i * kDB + tb * 4);
        const float sa[4] = {va.x, va.y, va.z, va.w};
        const float2 z01 = make_float2(vb.x, vb.y), z23 = make_float2(vb.z, vb.w);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float2 s2 = make_float2(sa[r], sa[r]);
          w2[r][0] = __ffma2_rn(s2, z01, w2[r][0]);
          w2[r][1] = __ffma2_rn(s2, z23, w2[r][1]);
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        w[r][0] = w2[r][0].x;
        w[r][1] = w2[r][0].y;
        w[r][2] = w2[r][1].x;
        w[r][3] = w2[r][1].y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) w[r][c] = T(0);
#pragma unroll 5
      for (int i = 0; i < l; ++i) {
        T sa[4], zb[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) sa[r] = Ss[i * kDA + ta * 4 + r];
#pragma unroll
        for (int c = 0; c < 4; ++c) zb[c] = Zs[i * kDB + tb * 4 + c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) w[r][c] = fma(sa[r], zb[c], w[r][c]);
      }
    }

    T acc[NA];
#pragma unroll
    for (int q = 0; q < NA; ++q) acc[q] = T(0);
    if constexpr (sizeof(T) == 4 && DP % 2 == 0) {
      // fp32: the d coordinate differences, their squares and the d lengthscale sums as paired
      // FADD2 / FFMA2 / FMUL2 over two coordinates (same products and sums per coordinate as below)
      float2 acc2[DP / 2];
#pragma unroll
      for (int k = 0; k < DP / 2; ++k) acc2[k] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int bl = tb * 4 + c;
        float2 xb2[DP / 2];
#pragma unroll
        for (int k = 0; k < DP / 2; ++k) xb2[k] = *reinterpret_cast<const float2*>(Xb + bl * DP + 2 * k);
        const float ub = Ub[bl];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int al = ta * 4 + r;
          float2 df[DP / 2];
          float2 s2 = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int k = 0; k < DP / 2; ++k) {
            const float2 xa2 = *reinterpret_cast<const float2*>(Xa + al * DP + 2 * k);
            df[k] = __fadd2_rn(xa2, make_float2(-xb2[k].x, -xb2[k].y));
            s2 = __ffma2_rn(df[k], df[k], s2);
          }
          float e, ds;
          shape_pair<float, FAM>(s2.x + s2.y, e, ds);
          const float q = fmaf(-cmix, w[r][c], Ua[al] * ub);  // u_a u_b - (n/l) W_ab
          acc[0] = fmaf(e, q, acc[0]);
          const float g = ds * q;
          const float2 g2 = make_float2(g, g);
#pragma unroll
          for (int k = 0; k < DP / 2; ++k) acc2[k] = __ffma2_rn(__fmul2_rn(g2, df[k]), df[k], acc2[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < DP / 2; ++k) {
        acc[1 + 2 * k] = acc2[k].x;
        acc[2 + 2 * k] = acc2[k].y;
      }
    } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int bl = tb * 4 + c;
      T xb[DP];
#pragma unroll
      for (int k = 0; k < DP; ++k) xb[k] = Xb[bl * DP + k];
      const T ub = Ub[bl];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int al = ta * 4 + r;
        T dd[DP];
        T s = T(0);
#pragma unroll
        for (int k = 0; k < DP; ++k) {
          const T df = Xa[al * DP + k] - xb[k];
          dd[k] = df * df;
          s += dd[k];
        }
        T e, ds;
        shape_pair<T, FAM>(s, e, ds);
        const T q = fma(-cmix, w[r][c], Ua[al] * ub);  // u_a u_b - (n/l) W_ab
        acc[0] = fma(e, q, acc[0]);
        const T g = ds * q;
#pragma unroll
        for (int k = 0; k < DP; ++k) acc[1 + k] = fma(g, dd[k], acc[1 + k]);
      }
    }
    }
#pragma unroll
    for (int q = 0; q < NA; ++q) acc64[q] += static_cast<double>(acc[q]);
    __syncthreads();  // buffer buf is restaged by the next iteration
  }

  // fixed-order block reduction -> one partial row per CTA
  const long long blk = static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x;
  for (int q = 0; q < NA; ++q) {
    const double v = block_sum(acc64[q], red);
    if (tid == 0) partials[blk * NA + q] = v;
  }
}

template <typename T, int FAM, int DP>
static cudaError_t launch_dc_t(const void* X, const void* U, const void* S, const void* Z, int n_pad, int l,
                               int a_begin, int a_rows, double cmix, double* partials, int* nblocks,
                               cudaStream_t st) {
  const size_t sm = sizeof(T) * (static_cast<size_t>(l) * kDA + kDA * DP + kDA +
                                 2 * (static_cast<size_t>(l) * kDB + kDB * DP + kDB));
  auto k = deriv_contract_kernel<T, FAM, DP>;
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    if (e != cudaSuccess) return e;
  }
  const int nat = (a_rows + kDA - 1) / kDA;
  const int nbt = n_pad / kDB;
  dim3 g(nat, (nbt + kDBTilesPerBlock - 1) / kDBTilesPerBlock);
  *nblocks = static_cast<int>(g.x * g.y);
  if (partials == nullptr) return cudaSuccess;  // size query
  k<<<g, kDThreads, sm, st>>>(static_cast<const T*>(X), static_cast<const T*>(U), static_cast<const T*>(S),
                              static_cast<const T*>(Z), n_pad, l, a_begin, static_cast<T>(cmix), partials);
  return cudaGetLastError();
}

template <typename T, int FAM>
static cudaError_t launch_dc_dp(int dp, const void* X, const void* U, const void* S, const void* Z, int n_pad, int l,
                                int a_begin, int a_rows, double cmix, double* partials, int* nblocks,
                                cudaStream_t st) {
  switch (dp) {
    case 4: return launch_dc_t<T, FAM, 4>(X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
    case 12: return launch_dc_t<T, FAM, 12>(X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
    case 20: return launch_dc_t<T, FAM, 20>(X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
    case 32: return launch_dc_t<T, FAM, 32>(X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
static cudaError_t launch_dc_fam(int fam, int dp, const void* X, const void* U, const void* S, const void* Z,
                                 int n_pad, int l, int a_begin, int a_rows, double cmix, double* partials,
                                 int* nblocks, cudaStream_t st) {
  switch (fam) {
    case kRBF: return launch_dc_dp<T, kRBF>(dp, X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
    case kMatern12: return launch_dc_dp<T, kMatern12>(dp, X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
    case kMatern32: return launch_dc_dp<T, kMatern32>(dp, X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
    case kMatern52: return launch_dc_dp<T, kMatern52>(dp, X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
  }
  return cudaErrorInvalidValue;
}

// U/S/Z layout: U [n_pad], S and Z column-major [l][n_pad]; X [n_pad][dp].
cudaError_t launch_deriv_contract(bool fp64, int family, int dp, const void* X, const void* U, const void* SZ,
                                  int a_begin, int a_rows, int n_pad, int l, double cmix, double* partials,
                                  int* nblocks, cudaStream_t st) {
  const size_t elem = fp64 ? 8 : 4;
  const void* S = SZ;
  const void* Z = static_cast<const unsigned char*>(SZ) + elem * static_cast<size_t>(l) * n_pad;
  return fp64 ? launch_dc_fam<double>(family, dp, X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st)
              : launch_dc_fam<float>(family, dp, X, U, S, Z, n_pad, l, a_begin, a_rows, cmix, partials, nblocks, st);
}

}  // namespace gpk
