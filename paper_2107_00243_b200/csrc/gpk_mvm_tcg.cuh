// Tensor-core fused kernel MVM, "Gram" variant: BOTH contractions on tcgen05.
//
//   out[:, c] = scale * sum_j k(x_i, x_j) V[j, c]
//
// The squared distances come from the expanded form the reference itself uses
// for its kernel columns (kernels.hpp:166-168, 235-243):
//     s_ij = |x_i|^2 + |x_j|^2 - 2 x_i . x_j
// with the cross term x_i . x_j computed on the tensor cores in split precision
// (3xTF32) from coordinates centred on their mean (distances are translation
// invariant; centring keeps |x|^2 small so the cancellation error stays at the
// level of the fp32 direct-difference path — the host enables this kernel only
// when max |x|^2 of the centred, pre-scaled coordinates is below a bound, and
// never for Matern-1/2 whose value is not smooth in s at s = 0).  Near pairs
// (s <= (|x_i|^2 + |x_j|^2)/16, the diagonal included), where the cancellation
// would dominate, are recomputed from fp32 direct differences.  The CUDA cores then only evaluate the
// kernel shape (MUFU sqrt / ex2) and split it into tf32 hi/lo for the second
// tensor-core contraction with V (as in gpk_mvm_tc.cuh).
//
// Both A operands live in TENSOR MEMORY (tcgen05.mma with [a] in TMEM): the
// CTA's coordinate block A_x (written once by the producers) and each kernel
// tile K_tile (written by the producers with tcgen05.st instead of st.shared),
// so shared memory only feeds the small B operands (X_j, V_j).  TMEM columns:
// [0,64) two Gram tiles | [64,128) A_x hi/lo | [128,256) two K_tile hi/lo
// stages | [256, 256+2 NPAD) two accumulator buffers.
//
// CTA = 128 output rows x NPAD columns, j-tiles of 32:
//   warp 0     : TMA producer — per tile the pre-swizzled X_j hi/lo tile,
//                |x_j|^2 and the V_j hi/lo tiles
//   warp 1     : TMEM allocator + single-thread MMA issuer.  Per tile:
//                G = A_x X_j^T (M=128, N=32, 3 x KS instructions) into a double-
//                buffered TMEM Gram tile, issued one tile AHEAD of
//                Acc += K_tile V_j (M=128, N=NPAD, 12 instructions)
//   warps 2..17: 16 producer warps: tcgen05.ld 8 Gram values per thread, kernel
//                shape, tf32 split, 128B-swizzled A tile; fp64 drain of TMEM.
#pragma once
#include "gpk_mvm_tc.cuh"

namespace gpk {
namespace tcg {

using tc::AS;
using tc::ATILE;
using tc::BK;
using tc::BM;
using tc::JPT;
using tc::NPW;
using tc::RPT;
using tc::S;
using tc::THREADS;

constexpr uint32_t XG_TILE = 32 * 32 * 4;  // one 32-row x 32-coordinate tf32 tile (hi or lo), 4 KB
constexpr int SG = 4;  // X_j / V_j stages
#ifdef GPK_TCG_TRACE  // experiment: per-tile clock64 stamps of CTA (0,0) -> gpk_tcg_trace
__device__ long long g_tcg_trace[8 * 1024];
#define GPK_TRACE(slot, it) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && (it) < 1000) g_tcg_trace[(slot) * 1024 + (it)] = clock64();
#else
#define GPK_TRACE(slot, it)
#endif
#ifdef GPK_TCG_SPIN_ISSUER  // experiment switch: single-thread issuers poll instead of suspending
#define GPK_ISSUER_WAIT mbar_wait
#else
#define GPK_ISSUER_WAIT mbar_wait_sleep
#endif
#ifdef GPK_TCG_SPIN_PRODUCER
#define GPK_PRODUCER_WAIT mbar_wait
#else
#define GPK_PRODUCER_WAIT mbar_wait_sleep
#endif
// TMEM column map
constexpr uint32_t T_GRAM = 0, T_AX = 64, T_AT = 128, T_ACC = 256;

GPK_DEV void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
GPK_DEV void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
// one lane of a converged warp (the tcgen05 issue idiom: the warp runs the control
// flow and waits together, one elected lane issues; keeps operands in uniform registers)
GPK_DEV uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred;
}
GPK_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

GPK_DEV float2 f2_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
constexpr float kGuard = 1.0f / 16.0f;  // cancellation guard (see the producer loop)

template <int FAM, int KS, int NC8>
__global__ void __launch_bounds__(THREADS, 1)
    fused_kmvm_tcg_kernel(const float* __restrict__ Xh, const float* __restrict__ Xl, const float* __restrict__ Xn,
                          const float* __restrict__ X32, const float* __restrict__ Vhi, const float* __restrict__ Vlo, double* __restrict__ out,
                          MvmArgs a) {
  constexpr int NPAD = 8 * NC8;
  constexpr uint32_t VTILE = NPAD * BK * 4;
  constexpr int HC = (NC8 + RPT - 1) / RPT;
  constexpr uint32_t TMEM_COLS = 512;
  constexpr uint32_t ACC0 = T_ACC;

  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* sbase = smem_raw + (base - raw);
  // carve: Bx[SG][2] | V[SG][2] | N[SG] | barriers | tmem slot
  const uint32_t sBx = base;
  const uint32_t sV = sBx + SG * 2 * XG_TILE;
  const uint32_t sN = sV + SG * 2 * VTILE;
  const float* Ns = reinterpret_cast<const float*>(sbase + (sN - base));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + (sN - base) + SG * 128);
  uint64_t* xv_full = bars;
  uint64_t* xv_empty = bars + SG;
  uint64_t* a_full = bars + 2 * SG;
  uint64_t* a_empty = bars + 2 * SG + AS;
  uint64_t* g_full = bars + 2 * SG + 2 * AS;
  uint64_t* g_empty = g_full + 2;
  uint64_t* acc_full = g_full + 4;
  uint64_t* acc_empty = g_full + 6;
  uint64_t* ax_ready = g_full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(g_full + 9);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int row0 = a.row_begin + blockIdx.x * BM;
  const int jt0 = blockIdx.y * a.jtiles_per_split;
  const int jt1 = min(jt0 + a.jtiles_per_split, a.n_pad / BK);
  const int nt = jt1 - jt0;
  const int F = a.flush > 0 ? a.flush : 1;
  if (threadIdx.x == 0) GPK_TRACE(0, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < SG; ++s) {
      mbar_init(&xv_full[s], 1);
      mbar_init(&xv_empty[s], 1);
    }
    for (int s = 0; s < AS; ++s) {
      mbar_init(&a_full[s], NPW);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&g_full[s], 1);
      mbar_init(&g_empty[s], NPW);
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], NPW);
    }
    mbar_init(ax_ready, NPW);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) GPK_TRACE(0, 1);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0 && nt > 0) {
      for (int it = 0; it < nt; ++it) {
        const int s = it % SG;
        GPK_ISSUER_WAIT(&xv_empty[s], ((it / SG) & 1) ^ 1);
        const long long jt = jt0 + it;
#ifdef GPK_TCG_NO_LOAD
        if (it >= SG) { tc::mbar_arrive(&xv_full[s]); continue; }
#endif
        mbar_arrive_expect_tx(&xv_full[s], 2 * XG_TILE + 128 + 2 * VTILE);
        bulk_g2s(sbase + (sBx - base) + (s * 2 + 0) * XG_TILE, Xh + jt * 1024, XG_TILE, &xv_full[s]);
        bulk_g2s(sbase + (sBx - base) + (s * 2 + 1) * XG_TILE, Xl + jt * 1024, XG_TILE, &xv_full[s]);
        bulk_g2s(sbase + (sN - base) + s * 128, Xn + jt * 32, 128, &xv_full[s]);
        bulk_g2s(sbase + (sV - base) + (s * 2 + 0) * VTILE, Vhi + jt * NPAD * BK, VTILE, &xv_full[s]);
        bulk_g2s(sbase + (sV - base) + (s * 2 + 1) * VTILE, Vlo + jt * NPAD * BK, VTILE, &xv_full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp converged, elected lane issues) ----------------
    if (nt > 0) {
      constexpr uint32_t idesc_v = tc::idesc_tf32(NPAD);
      constexpr uint32_t idesc_g = tc::idesc_tf32(32);
      GPK_ISSUER_WAIT(ax_ready, 0);
      auto gram = [&](int k) {
        const int s = k % SG, gb = k & 1;
        GPK_ISSUER_WAIT(&xv_full[s], (k / SG) & 1);
        GPK_ISSUER_WAIT(&g_empty[gb], ((k >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t bh = sBx + (s * 2 + 0) * XG_TILE, bl = sBx + (s * 2 + 1) * XG_TILE;
        if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint32_t ko = ks * 32;
          const uint32_t tah = tmem_base + T_AX + ks * 8, tal = tmem_base + T_AX + 32 + ks * 8;
          const uint64_t dbh = tc::smem_desc_sw128(bh + ko), dbl = tc::smem_desc_sw128(bl + ko);
          mma_tf32_ts(tmem_base + T_GRAM + gb * 32, tah, dbh, idesc_g, ks > 0 ? 1u : 0u);
          mma_tf32_ts(tmem_base + T_GRAM + gb * 32, tah, dbl, idesc_g, 1u);
          mma_tf32_ts(tmem_base + T_GRAM + gb * 32, tal, dbh, idesc_g, 1u);
        }
        tc::tc_commit(&g_full[gb]);
        }
        __syncwarp();
        if (lane == 0) GPK_TRACE(7, k);
      };
      gram(0);
      for (int it = 0; it < nt; ++it) {
        if (it + 1 < nt) gram(it + 1);  // the next Gram tile overlaps this tile's kernel-shape evaluation
        const int s = it % SG, as = it % AS;
        const int g = it / F, buf = g & 1;
        if (it % F == 0) GPK_ISSUER_WAIT(&acc_empty[buf], ((g >> 1) & 1) ^ 1);
        GPK_ISSUER_WAIT(&a_full[as], (it / AS) & 1);
        if (lane == 0) GPK_TRACE(3, it);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + ACC0 + buf * NPAD;
        const uint32_t tah = tmem_base + T_AT + as * 64, tal = tah + 32;
        const uint32_t bhi = sV + (s * 2 + 0) * VTILE, blo = sV + (s * 2 + 1) * VTILE;
        if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint32_t koff = ks * 32;
          const uint64_t dbh = tc::smem_desc_sw128(bhi + koff), dbl = tc::smem_desc_sw128(blo + koff);
          const uint32_t acc = (it % F != 0 || ks > 0) ? 1u : 0u;
          mma_tf32_ts(d_tmem, tah + ks * 8, dbh, idesc_v, acc);
          mma_tf32_ts(d_tmem, tah + ks * 8, dbl, idesc_v, 1u);
          mma_tf32_ts(d_tmem, tal + ks * 8, dbh, idesc_v, 1u);
        }
        tc::tc_commit(&a_empty[as]);
        tc::tc_commit(&xv_empty[s]);  // also covers the Gram MMA of this stage and the producers' norm reads
        if (it % F == F - 1 || it == nt - 1) tc::tc_commit(&acc_full[buf]);
        }
        __syncwarp();
        if (lane == 0) GPK_TRACE(6, it);
      }
    }
  } else {
    // ---------------- producer / epilogue warps ----------------
    const int pw = warp - 2;
    const int lg = warp & 3;   // TMEM lane group
    const int q = pw >> 2;     // 8-column slice of the j-tile, and column-chunk subset of the drain
    const int r = lg * 32 + lane;
    const int row = row0 + r;
    const float ni = Xn[row];
    const float2 ni2 = make_float2(ni, ni);
    const uint32_t tlane = static_cast<uint32_t>(lg * 32) << 16;
    {  // this row's centred coordinates (tf32 hi / lo, columns q*8 .. q*8+7) -> A_x in TMEM
      const long long tb = static_cast<long long>(row >> 5) * 1024;
      const int rr = row & 31;
      float h8[8], l8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = q * 8 + u;
        const long long off = tb + (rr >> 3) * 256 + (rr & 7) * 32 + ((((k >> 2) ^ (rr & 7))) << 2) + (k & 3);
        h8[u] = Xh[off];
        l8[u] = Xl[off];
      }
      tmem_st8(tmem_base + tlane + T_AX + q * 8, h8);
      tmem_st8(tmem_base + tlane + T_AX + 32 + q * 8, l8);
      tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(ax_ready);
    }
    double acc64[HC * 8];
#pragma unroll
    for (int e = 0; e < HC * 8; ++e) acc64[e] = 0.0;
    auto drain = [&](int g) {
      const int buf = g & 1;
      GPK_PRODUCER_WAIT(&acc_full[buf], (g >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int h = 0; h < HC; ++h) {
        const int c8 = q + h * RPT;
        if (c8 < NC8) {
          uint32_t v[8];
          tc::tmem_ld8(tmem_base + tlane + ACC0 + buf * NPAD + c8 * 8, v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) acc64[h * 8 + e] += static_cast<double>(__uint_as_float(v[e]));
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[buf]);
    };
    for (int it = 0; it < nt; ++it) {
      const int s = it % SG, as = it % AS, gb = it & 1;
      const int jb = (jt0 + it) * BK + q * JPT;  // global index of this thread's first column
      if (threadIdx.x == 64) GPK_TRACE(1, it);
      GPK_PRODUCER_WAIT(&g_full[gb], (it >> 1) & 1);
      if (threadIdx.x == 64) GPK_TRACE(2, it);
      tc::tc_fence_after();
      uint32_t gv[8];
      tc::tmem_ld8(tmem_base + tlane + T_GRAM + gb * 32 + q * JPT, gv);
      tc::tmem_wait_ld();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&g_empty[gb]);
      GPK_PRODUCER_WAIT(&xv_full[s], (it / SG) & 1);  // |x_j|^2 of this stage visible to the generic proxy
      const float4 n0 = reinterpret_cast<const float4*>(Ns + s * 32 + q * JPT)[0];
      const float4 n1 = reinterpret_cast<const float4*>(Ns + s * 32 + q * JPT)[1];
      const float2 nj[4] = {make_float2(n0.x, n0.y), make_float2(n0.z, n0.w), make_float2(n1.x, n1.y),
                            make_float2(n1.z, n1.w)};
      float sv[8];
      uint32_t near = 0;  // entries whose expanded-form value is within the cancellation guard
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float2 nn = f2_add(nj[p], ni2);
        const float2 g2 = make_float2(__uint_as_float(gv[2 * p]), __uint_as_float(gv[2 * p + 1]));
        const float2 t2 = __ffma2_rn(make_float2(-2.0f, -2.0f), g2, nn);
        sv[2 * p] = fmaxf(t2.x, 0.0f);
        sv[2 * p + 1] = fmaxf(t2.y, 0.0f);
        near |= (sv[2 * p] <= kGuard * nn.x ? 1u : 0u) << (2 * p);
        near |= (sv[2 * p + 1] <= kGuard * nn.y ? 1u : 0u) << (2 * p + 1);
      }
      // Cancellation guard: s <= (|x_i|^2 + |x_j|^2) / 16 (near pairs, incl. the
      // diagonal) is recomputed from fp32 direct differences of the un-centred
      // coordinates, so the expanded form only serves pairs whose relative error in s
      // stays at the fp32 level.  Rare for the spread-out data auto mode selects.
#ifdef GPK_TCG_NO_GUARD
      near = 0;
#endif
      if (__any_sync(0xffffffffu, near != 0)) {
#pragma unroll 1
        for (int u = 0; u < JPT; ++u) {
          if (near & (1u << u)) {
            const float4* xi = reinterpret_cast<const float4*>(X32 + static_cast<long long>(row) * a.dp);
            const float4* xj = reinterpret_cast<const float4*>(X32 + static_cast<long long>(jb + u) * a.dp);
            float acc = 0.0f;
            for (int k = 0; k < a.dp / 4; ++k) {
              const float4 p = xi[k], q4 = xj[k];
              const float d0 = p.x - q4.x, d1 = p.y - q4.y, d2 = p.z - q4.z, d3 = p.w - q4.w;
              acc = fmaf(d0, d0, acc);
              acc = fmaf(d1, d1, acc);
              acc = fmaf(d2, d2, acc);
              acc = fmaf(d3, d3, acc);
            }
            sv[u] = acc;
          }
        }
      }
      GPK_PRODUCER_WAIT(&a_empty[as], ((it / AS) & 1) ^ 1);
      float eh[8], el[8];
#pragma unroll
      for (int u = 0; u < JPT; ++u) {
        const float e = kval32<FAM>(sv[u]);
        eh[u] = tc::to_tf32_alu(e);
        el[u] = e - eh[u];
      }
#ifndef GPK_TCG_NO_STORE
      tmem_st8(tmem_base + tlane + T_AT + as * 64 + q * JPT, eh);
      tmem_st8(tmem_base + tlane + T_AT + as * 64 + 32 + q * JPT, el);
#endif
      tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&a_full[as]);
      if (lane == 0 && it < 64) GPK_TRACE(4, it * 16 + pw);
      if (it % F == 0 && it > 0) drain(it / F - 1);
    }
    if (nt > 0) drain((nt - 1) / F);
    if (threadIdx.x == 64) GPK_TRACE(0, 2);
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
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

template <int NC8>
constexpr size_t tcg_smem_bytes() {
  return 1024 + SG * 2 * XG_TILE + SG * 2 * (8 * NC8 * BK * 4) + SG * 128 + (2 * SG + 2 * AS + 9) * 8 + 16;
}

template <int FAM, int KS, int NC8>
cudaError_t launch_tcg_t(const float* Xh, const float* Xl, const float* Xn, const float* X32, const float* Vhi, const float* Vlo,
                         double* out, const MvmArgs& a, dim3 grid, cudaStream_t st) {
  constexpr size_t sm = tcg_smem_bytes<NC8>();
  static_assert(sm <= 232448, "tcg smem");
  auto k = fused_kmvm_tcg_kernel<FAM, KS, NC8>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k<<<grid, THREADS, sm, st>>>(Xh, Xl, Xn, X32, Vhi, Vlo, out, a);
  return cudaGetLastError();
}

template <int FAM>
cudaError_t launch_tcg_fam(int ks, int nc8, const float* Xh, const float* Xl, const float* Xn, const float* X32,
                           const float* Vhi,
                           const float* Vlo, double* out, const MvmArgs& a, dim3 g, cudaStream_t st) {
#define GPK_TCG_NC(N)                                                                 \
  case N:                                                                             \
    switch (ks) {                                                                     \
      case 1: return launch_tcg_t<FAM, 1, N>(Xh, Xl, Xn, X32, Vhi, Vlo, out, a, g, st);    \
      case 2: return launch_tcg_t<FAM, 2, N>(Xh, Xl, Xn, X32, Vhi, Vlo, out, a, g, st);    \
      case 3: return launch_tcg_t<FAM, 3, N>(Xh, Xl, Xn, X32, Vhi, Vlo, out, a, g, st);    \
      case 4: return launch_tcg_t<FAM, 4, N>(Xh, Xl, Xn, X32, Vhi, Vlo, out, a, g, st);    \
      default: return cudaErrorInvalidValue;                                          \
    }
  switch (nc8) {
    GPK_TCG_NC(1) GPK_TCG_NC(2) GPK_TCG_NC(4) GPK_TCG_NC(6) GPK_TCG_NC(7) GPK_TCG_NC(8) GPK_TCG_NC(9)
    GPK_TCG_NC(10) GPK_TCG_NC(12) GPK_TCG_NC(16)
    default: break;
  }
#undef GPK_TCG_NC
  return cudaErrorInvalidValue;
}

}  // namespace tcg
}  // namespace gpk

#define GPK_INSTANTIATE_TCG_FAMILY(FAM)                                                                         \
  namespace gpk {                                                                                               \
  namespace tcg {                                                                                               \
  template cudaError_t launch_tcg_fam<FAM>(int, int, const float*, const float*, const float*, const float*,   \
                                           const float*, \
                                           const float*, double*, const MvmArgs&, dim3, cudaStream_t);          \
  }                                                                                                             \
  }
