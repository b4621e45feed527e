// Tensor-core (tcgen05) variant of the fused kernel MVM.
//
//   out[:, c] = scale * sum_j k(x_i, x_j) V[j, c]
//
// Kernel entries are produced on the CUDA cores exactly as in the SIMT kernel
// (fp32 direct-difference distances, MUFU ex2/sqrt); the contraction K_tile x
// V_tile runs on the 5th-generation tensor cores in split precision
// ("3xTF32": a = a_hi + a_lo, a*b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi, with
// a_hi/a_lo rounded to tf32 by cvt.rna), accumulating in TMEM (fp32) over
// flush groups of 4 j-tiles (128 entries) that the producer warps drain into
// fp64 registers.
//
// CTA = 128 output rows x NPAD (= 8*NC8) columns, j-tiles of 32:
//   warp 0      : TMA producer — cp.async.bulk of X_j [32 x DP] and the
//                 pre-swizzled V_j^T hi/lo tiles [NPAD x 32] into a 3-stage ring
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer
//                 (M=128, N=NPAD, K=8 per instruction, 12 instructions per tile)
//   warps 2..17 : 16 producer warps: 4 threads per row, 8 entries each per tile,
//                 written as tf32 hi/lo into a double-buffered 128B-swizzled
//                 K-major A tile; then fp64 drain of their TMEM lane group.
// Synchronisation: mbarriers (TMA complete_tx, producer arrivals, tcgen05.commit).
#pragma once
#include "gpk_common.cuh"
#include "gpk_internal.h"
#include "gpk_mvm.cuh"

namespace gpk {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int S = 3;       // X/V stages
constexpr int AS = 2;      // A-tile stages
// tiles per TMEM flush group: MvmArgs::flush (runtime; 1..8)
constexpr int NPW = 16;    // producer warps
constexpr int RPT = NPW / 4;              // producer threads per row
constexpr int JPT = BK / RPT;             // entries per producer thread per tile (8)
constexpr int THREADS = (2 + NPW) * 32;   // 576
constexpr uint32_t ATILE = BM * BK * 4;   // 16 KB per hi/lo A tile

// --------------------------------------------------------------------------
// tcgen05 / TMEM / mbarrier PTX
// --------------------------------------------------------------------------
GPK_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
GPK_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
GPK_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
GPK_DEV void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
GPK_DEV void tc_mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
GPK_DEV void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
GPK_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
GPK_DEV float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// paired fp32 (sm_100 FADD2 / FFMA2): two lanes of work per issue slot.  The
// intrinsics are required: inline-asm f32x2 on 64-bit registers is split by
// ptxas into scalar FADD/FFMA.
GPK_DEV float2 f2_sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
GPK_DEV float2 f2_fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
GPK_DEV float f2_hsum(float2 a) { return a.x + a.y; }
// round-to-nearest (ties away) to tf32 with integer ALU ops instead of the
// quarter-rate conversion unit (finite inputs)
GPK_DEV float to_tf32_alu(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
GPK_DEV void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// K-major operand, 128B swizzle (canonical UMMA layout: 8-row atoms of 1024 B,
// SBO = 1024 B between atoms, LBO unused (=16 B), version 1 for sm_100).
GPK_DEV uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;            // LBO (16 B units)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO
  d |= static_cast<uint64_t>(1) << 46;            // descriptor version (Blackwell)
  d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, K-major both, N, M = 128
__host__ __device__ constexpr uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

// byte offset of element (row r, k) in a 128B-swizzled K-major tile of 32 fp32 per row
GPK_DEV uint32_t sw128_off(int r, int k) {
  return static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ (r & 7))) << 4) + ((k & 3) << 2));
}

template <int FAM, int DP, int NC8>
__global__ void __launch_bounds__(THREADS, 1)
    fused_kmvm_tc_kernel(const float* __restrict__ X, const float* __restrict__ Vhi, const float* __restrict__ Vlo,
                         double* __restrict__ out, MvmArgs a) {
  constexpr int NPAD = 8 * NC8;
  constexpr uint32_t VTILE = NPAD * BK * 4;     // bytes per hi or lo V tile
  constexpr uint32_t XTILE = BK * DP * 4;
  constexpr int HC = (NC8 + RPT - 1) / RPT;     // max 8-column chunks drained per thread
  constexpr uint32_t TMEM_COLS = (2 * NPAD <= 32) ? 32 : (2 * NPAD <= 64) ? 64 : (2 * NPAD <= 128) ? 128 : 256;

  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* sbase = smem_raw + (base - raw);
  // carve: A[AS][2] | V[S][2] | X[S] | barriers | tmem slot
  const uint32_t sA = base;
  const uint32_t sV = sA + AS * 2 * ATILE;
  const uint32_t sX = sV + S * 2 * VTILE;
  float* Xs = reinterpret_cast<float*>(sbase + (sX - base));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + (sX - base) + S * XTILE);
  uint64_t* xv_full = bars;
  uint64_t* x_empty = bars + S;
  uint64_t* v_empty = bars + 2 * S;
  uint64_t* a_full = bars + 3 * S;
  uint64_t* a_empty = bars + 3 * S + AS;
  uint64_t* acc_full = bars + 3 * S + 2 * AS;
  uint64_t* acc_empty = bars + 3 * S + 2 * AS + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 2 * AS + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int row0 = a.row_begin + blockIdx.x * BM;
  const int jt0 = blockIdx.y * a.jtiles_per_split;
  const int jt1 = min(jt0 + a.jtiles_per_split, a.n_pad / BK);
  const int nt = jt1 - jt0;
  const int F = a.flush > 0 ? a.flush : 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&xv_full[s], 1);
      mbar_init(&x_empty[s], NPW);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < AS; ++s) {
      mbar_init(&a_full[s], NPW);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], NPW);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int it = 0; it < nt; ++it) {
        const int s = it % S;
        const uint32_t par = ((it / S) & 1) ^ 1;
        mbar_wait_sleep(&x_empty[s], par);
        mbar_wait_sleep(&v_empty[s], par);
        const long long jt = jt0 + it;
        mbar_arrive_expect_tx(&xv_full[s], XTILE + 2 * VTILE);
        bulk_g2s(sbase + (sX - base) + s * XTILE, X + jt * BK * DP, XTILE, &xv_full[s]);
        bulk_g2s(sbase + (sV - base) + (s * 2 + 0) * VTILE, Vhi + jt * NPAD * BK, VTILE, &xv_full[s]);
        bulk_g2s(sbase + (sV - base) + (s * 2 + 1) * VTILE, Vlo + jt * NPAD * BK, VTILE, &xv_full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(NPAD);
      for (int it = 0; it < nt; ++it) {
        const int s = it % S, as = it % AS;
        const int g = it / F, buf = g & 1;
        if (it % F == 0) mbar_wait_sleep(&acc_empty[buf], ((g >> 1) & 1) ^ 1);
        mbar_wait_sleep(&a_full[as], (it / AS) & 1);
        mbar_wait_sleep(&xv_full[s], (it / S) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * NPAD;
        const uint32_t ahi = sA + (as * 2 + 0) * ATILE, alo = sA + (as * 2 + 1) * ATILE;
        const uint32_t bhi = sV + (s * 2 + 0) * VTILE, blo = sV + (s * 2 + 1) * VTILE;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint32_t koff = ks * 32;  // 8 tf32 = 32 bytes along K
          const uint64_t dah = smem_desc_sw128(ahi + koff), dal = smem_desc_sw128(alo + koff);
          const uint64_t dbh = smem_desc_sw128(bhi + koff), dbl = smem_desc_sw128(blo + koff);
          const uint32_t acc = (it % F != 0 || ks > 0) ? 1u : 0u;
          tc_mma_tf32(d_tmem, dah, dbh, idesc, acc);
          tc_mma_tf32(d_tmem, dah, dbl, idesc, 1u);
          tc_mma_tf32(d_tmem, dal, dbh, idesc, 1u);
        }
        tc_commit(&a_empty[as]);
        tc_commit(&v_empty[s]);
        if (it % F == F - 1 || it == nt - 1) tc_commit(&acc_full[buf]);
      }
    }
  } else {
    // ---------------- producer / epilogue warps ----------------
    const int pw = warp - 2;           // 0..15
    const int lg = warp & 3;           // TMEM lane group this warp may access
    const int q = pw >> 2;             // quarter: j-range and column-chunk subset
    const int r = lg * 32 + lane;      // row within the tile == TMEM lane
    const int row = row0 + r;
    float2 xr[DP / 2];  // this row's coordinates, packed in pairs
#pragma unroll
    for (int k = 0; k < DP / 4; ++k) {
      const float4 v = reinterpret_cast<const float4*>(X + static_cast<long long>(row) * DP)[k];
      xr[2 * k] = make_float2(v.x, v.y);
      xr[2 * k + 1] = make_float2(v.z, v.w);
    }
    double acc64[HC * 8];
#pragma unroll
    for (int e = 0; e < HC * 8; ++e) acc64[e] = 0.0;
    // column chunks drained by this thread: c8 = q, q + RPT, ...
    auto drain = [&](int g) {
      const int buf = g & 1;
      mbar_wait_sleep(&acc_full[buf], (g >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < HC; ++h) {
        const int c8 = q + h * RPT;
        if (c8 < NC8) {
          uint32_t v[8];
          tmem_ld8(tmem_base + (static_cast<uint32_t>(lg * 32) << 16) + buf * NPAD + c8 * 8, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) acc64[h * 8 + e] += static_cast<double>(__uint_as_float(v[e]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    };
    for (int it = 0; it < nt; ++it) {
      const int s = it % S, as = it % AS;
      mbar_wait_sleep(&xv_full[s], (it / S) & 1);
      mbar_wait_sleep(&a_empty[as], ((it / AS) & 1) ^ 1);
      const float* xs = Xs + s * (BK * DP);
      const uint32_t ahi = sA + (as * 2 + 0) * ATILE, alo = sA + (as * 2 + 1) * ATILE;
#pragma unroll
      for (int c4 = 0; c4 < JPT / 4; ++c4) {
        float eh[4], el[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = q * JPT + c4 * 4 + u;
          const float4* xj = reinterpret_cast<const float4*>(xs + j * DP);
          float2 a0 = make_float2(0.f, 0.f), a1 = a0;  // four partial sums of squared differences
#pragma unroll
          for (int k = 0; k < DP / 4; ++k) {
            const float4 v = xj[k];
            const float2 d0 = f2_sub(xr[2 * k], make_float2(v.x, v.y));
            const float2 d1 = f2_sub(xr[2 * k + 1], make_float2(v.z, v.w));
            a0 = f2_fma(d0, d0, a0);
            a1 = f2_fma(d1, d1, a1);
          }
          const float e = kval32<FAM>(f2_hsum(a0) + f2_hsum(a1));
          eh[u] = to_tf32_alu(e);
          el[u] = e - eh[u];  // exact; the tensor core reads its leading tf32 bits
        }
        const uint32_t off = sw128_off(r, q * JPT + c4 * 4);
        st_shared_v4(ahi + off, eh[0], eh[1], eh[2], eh[3]);
        st_shared_v4(alo + off, el[0], el[1], el[2], el[3]);
      }
      fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&a_full[as]);
        mbar_arrive(&x_empty[s]);
      }
      if (it % F == 0 && it > 0) drain(it / F - 1);
    }
    if (nt > 0) drain((nt - 1) / F);
    // epilogue: column-major fp64 output (or split-K partial)
    if (row < a.row_end) {
      double* o = out + static_cast<long long>(blockIdx.y) * a.split_stride;
#pragma unroll
      for (int h = 0; h < HC; ++h) {
        const int c8 = q + h * RPT;
        if (c8 >= NC8) continue;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int col = c8 * 8 + e;
          if (col < a.t) o[static_cast<long long>(col) * a.ldo + (row - a.row_begin)] = a.scale * acc64[h * 8 + e];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

template <int NC8, int DP>
constexpr size_t tc_smem_bytes() {
  return 1024 /* alignment slack */ + AS * 2 * ATILE + S * 2 * (8 * NC8 * BK * 4) + S * (BK * DP * 4) +
         (3 * S + 2 * AS + 4) * 8 + 16;
}

template <int FAM, int DP, int NC8>
cudaError_t launch_tc_t(const float* X, const float* Vhi, const float* Vlo, double* out, const MvmArgs& a, dim3 grid,
                        cudaStream_t st) {
  constexpr size_t sm = tc_smem_bytes<NC8, DP>();
  auto k = fused_kmvm_tc_kernel<FAM, DP, NC8>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k<<<grid, THREADS, sm, st>>>(X, Vhi, Vlo, out, a);
  return cudaGetLastError();
}

template <int FAM>
cudaError_t launch_tc_fam(int dp, int nc8, const float* X, const float* Vhi, const float* Vlo, double* out,
                          const MvmArgs& a, dim3 g, cudaStream_t st) {
#define GPK_TC_NC(N)                                                          \
  case N:                                                                     \
    switch (dp) {                                                             \
      case 4: return launch_tc_t<FAM, 4, N>(X, Vhi, Vlo, out, a, g, st);      \
      case 12: return launch_tc_t<FAM, 12, N>(X, Vhi, Vlo, out, a, g, st);    \
      case 20: return launch_tc_t<FAM, 20, N>(X, Vhi, Vlo, out, a, g, st);    \
      case 32: return launch_tc_t<FAM, 32, N>(X, Vhi, Vlo, out, a, g, st);    \
      default: return cudaErrorInvalidValue;                                  \
    }
  switch (nc8) {
    GPK_TC_NC(1) GPK_TC_NC(2) GPK_TC_NC(4) GPK_TC_NC(6) GPK_TC_NC(7) GPK_TC_NC(8) GPK_TC_NC(9) GPK_TC_NC(10)
    GPK_TC_NC(12) GPK_TC_NC(16)
    default: break;
  }
#undef GPK_TC_NC
  return cudaErrorInvalidValue;
}

}  // namespace tc
}  // namespace gpk

#define GPK_INSTANTIATE_TC_FAMILY(FAM)                                                                          \
  namespace gpk {                                                                                               \
  namespace tc {                                                                                                \
  template cudaError_t launch_tc_fam<FAM>(int, int, const float*, const float*, const float*, double*,         \
                                          const MvmArgs&, dim3, cudaStream_t);                                 \
  }                                                                                                             \
  }
