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
// would dominate, are recomputed from fp32 direct differences.
//
// The CUDA cores then only evaluate the kernel shape (MUFU sqrt / ex2).  The
// entries are scaled by 2^10 and split into fp16 hi + lo; V is scaled per column
// by a power of two sigma_c (|V sigma| < 2^14) and split the same way, and
// K_tile V_j runs as three kind::f16 products (hi hi + hi lo + lo hi, fp32
// accumulate: 22 significant bits, the 3xTF32 level at twice the rate and half
// the instructions).  The output is rescaled by 1 / (2^10 sigma_c) in fp64.
//
// Both A operands live in TENSOR MEMORY (tcgen05.mma with [a] in TMEM): the
// CTA's coordinate block A_x (tf32 hi/lo, written once by the producers) and
// each kernel tile (packed fp16 pairs written with tcgen05.st), so shared memory
// only feeds the B operands (X_j, V_j).  TMEM columns:
//   [0,128) two 64-wide Gram tiles | [128,192) A_x hi/lo | [192,320) two kernel
//   tile stages (hi 32 + lo 32 packed columns) | [320, 320 + 2 NPAD) accumulators.
//
// CTA = 128 output rows x NPAD (<= 96) columns, j-tiles of 64:
//   warp 0     : TMA producer — per tile the pre-swizzled X_j hi/lo tile (64 x 32
//                tf32), |x_j|^2 and the V_j hi/lo tiles (NPAD x 64 fp16)
//   warp 1     : TMEM allocator + MMA issuer (converged warp, elected lane):
//                G = A_x X_j^T (M=128, N=64, 3 x KS tf32 instructions) issued one
//                tile AHEAD of Acc += K_tile V_j (M=128, N=NPAD, 4 x 3 f16 instructions)
//   warps 2, 3  : idle (register donors: setmaxnreg gives the producers 112 registers)
//   warps 4..19: 16 producer warps (TMEM lane group = warp % 4, 16-column slice of
//                the j-tile = (warp - 4) / 4): Gram -> distance -> kernel shape ->
//                fp16 hi/lo -> TMEM; fp64 drain of their accumulator lanes.
#pragma once
#include <cuda_fp16.h>

#include "gpk_mvm_tc.cuh"

namespace gpk {
namespace tcg {

constexpr int BM = 128;
constexpr int BK = 64;                    // j-tile
constexpr int NPW = 16;                   // producer warps
constexpr int RPT = 4;                    // producer warps per TMEM lane group
constexpr int JPT = BK / RPT;             // entries per producer thread per tile (16)
constexpr int THREADS = (4 + NPW) * 32;   // 640: warpgroup 0 = TMA issuer, MMA issuer, two idle register donors
// setmaxnreg: the 128 x (96 - 32) registers warpgroup 0 releases = the 512 x (112 - 96) the producers acquire
// (setmaxnreg.inc draws on the CTA's own released registers only)
constexpr int REGS_ISSUE = 32, REGS_PROD = 112;
constexpr int kConv = 4;                   // accumulation groups summed in fp32 (RN) per fp64 add
constexpr int SG = 4;                     // X_j / V_j stages
constexpr int AS = 2;                     // kernel-tile stages (TMEM)
constexpr int MAX_NPAD = 96;
constexpr uint32_t XG_TILE = BK * 32 * 4;  // 64 rows x 32 tf32 coordinates (hi or lo), 8 KB
constexpr uint32_t XJ_TILE = BK * 32 * 4;  // 64 fp32 coordinate rows (dp <= 32 each), guard path
constexpr uint32_t XI_BLOCK = BM * 32 * 4; // the CTA's 128 fp32 coordinate rows
constexpr uint32_t T_GRAM = 0, T_AX = 128, T_AT = 192, T_ACC = 320;
constexpr int kEntryLog2 = 10;             // entries scaled by 2^10: fp16 hi/lo stay normal
constexpr float kGuard = 1.0f / 16.0f;     // cancellation guard (see the producer loop)

#ifdef GPK_TCG_TRACE  // experiment: per-tile clock64 stamps of CTA (0,0) -> gpk_tcg_trace
__device__ long long g_tcg_trace[8 * 1024];
#define GPK_TRACE(slot, it) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && (it) < 1000) g_tcg_trace[(slot) * 1024 + (it)] = clock64();
#else
#define GPK_TRACE(slot, it)
#endif

GPK_DEV void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
               "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
               : "memory");
}
GPK_DEV void mma_ts_f16(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
               "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
               : "memory");
}
// instruction descriptor: D f32, A/B f16, K-major both, N, M = 128
__host__ __device__ constexpr uint32_t idesc_f16(int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}
GPK_DEV void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
GPK_DEV void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
GPK_DEV void tmem_st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
GPK_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// one lane of a converged warp (the tcgen05 issue idiom: the warp runs the control
// flow and waits together, one elected lane issues; operands stay in uniform registers)
GPK_DEV uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  return pred;
}
GPK_DEV uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
// fp16 hi / lo split of two entries: hi = f16(e) (packed, x in the low half), lo = f16(e - hi)
// with e - hi as ONE mixed-precision add per entry (FHADD: f32 = -f16 + f32) instead of
// unpacking hi to f32 first -- 4 instructions per 2 entries instead of 5.
GPK_DEV uint32_t split_f16x2(float2 e, uint32_t& lo) {
  uint32_t hb;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hb) : "f"(e.y), "f"(e.x));
  unsigned short hx = static_cast<unsigned short>(hb & 0xffffu), hy = static_cast<unsigned short>(hb >> 16);
  float lx, ly;
  asm("{\n\t.reg .f16 n;\n\tneg.f16 n, %1;\n\tadd.rn.f32.f16 %0, n, %2;\n\t}" : "=f"(lx) : "h"(hx), "f"(e.x));
  asm("{\n\t.reg .f16 n;\n\tneg.f16 n, %1;\n\tadd.rn.f32.f16 %0, n, %2;\n\t}" : "=f"(ly) : "h"(hy), "f"(e.y));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(ly), "f"(lx));
  return hb;
}

// DPD > 0: direct-difference mode (no Gram MMA): s_ij from the fp32 rows of X32 staged in
// shared memory (DPD = the padded coordinate count, <= 8) -- the low-dimensional / Matern-1/2
// path, sharing the pipeline, the fp16 split and the K_tile V_j contraction.
template <int FAM, int KS, int NC8, int DPD>
__global__ void __launch_bounds__(THREADS, 1)
    fused_kmvm_tcg_kernel(const float* __restrict__ Xh, const float* __restrict__ Xl, const float* __restrict__ Xn,
                          const float* __restrict__ X32, const __half* __restrict__ Vhi,
                          const __half* __restrict__ Vlo, const double* __restrict__ colscale,
                          double* __restrict__ out, MvmArgs a) {
  constexpr int NPAD = 8 * NC8;
  static_assert(NPAD <= MAX_NPAD, "NPAD");
  constexpr bool DIRECT = DPD > 0;
  static_assert(DPD % 4 == 0 && DPD <= 8, "DPD");
  constexpr uint32_t VTILE = NPAD * BK * 2;  // fp16 V_j tile (hi or lo)
  constexpr int HC = (NC8 + RPT - 1) / RPT;
  constexpr uint32_t TMEM_COLS = 512;

  // Gram mode: the A-side augmented image (row operand) follows the B-side one; the per-j-tile
  // norm maxima follow the norms (gram_pack_kernel)
  const float* XAh = Xh + static_cast<long long>(a.n_pad) * 32;
  const float* XAl = Xl + static_cast<long long>(a.n_pad) * 32;
  const float* Xtm = Xn + a.n_pad;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* sbase = smem_raw + (base - raw);
  // carve: Bx[SG][2] | V[SG][2] | N[SG] | barriers | tmem slot
  const uint32_t sBx = base;
  const uint32_t sV = sBx + SG * 2 * XG_TILE;
  const uint32_t sN = sV + SG * 2 * VTILE;
  const float* Ns = reinterpret_cast<const float*>(sbase + (sN - base));
  // fp32 coordinates for the cancellation guard: the j-tile rows per stage and the CTA's rows
  const uint32_t sXJ = sN + SG * BK * 4;
  const uint32_t sXI = sXJ + SG * XJ_TILE;
  const float* XJs = reinterpret_cast<const float*>(sbase + (sXJ - base));
  const float* XIs = reinterpret_cast<const float*>(sbase + (sXI - base));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + (sXI - base) + XI_BLOCK);
  uint64_t* xv_full = bars;
  uint64_t* xv_empty = bars + SG;
  uint64_t* a_full = bars + 2 * SG;
  uint64_t* a_empty = a_full + AS;
  uint64_t* g_full = a_empty + AS;
  uint64_t* g_empty = g_full + 2;
  uint64_t* acc_full = g_full + 4;
  uint64_t* acc_empty = g_full + 6;
  uint64_t* ax_ready = g_full + 8;
  uint64_t* xi_full = g_full + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(g_full + 10);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Work units: (row block, split) pairs u = rb * S + sp, the split a FIXED j-tile range (a
  // function of the global n), each unit's partial stored in its own split slot -- so the
  // sums never depend on which CTA runs a unit or on the shard.  CTA b runs the contiguous
  // units [b U / G, (b+1) U / G) of a persistent grid of G CTAs (G = U: one unit per CTA); a
  // row-block change inside a CTA is one CTA-wide barrier (the row tiles in TMEM / shared
  // memory are replaced only after every role has finished the previous row).
  const int ntiles = a.n_pad / BK;
  const int per = a.jtiles_per_split;
  const int S = (ntiles + per - 1) / per;
  const int nrb = (a.row_end - a.row_begin + BM - 1) / BM;
  const long long U = static_cast<long long>(nrb) * S;
  // Unit order (a.unit_order).  0: u = rb * S + sp, CTA b runs the CONTIGUOUS units [b U / G, (b+1) U / G) --
  // consecutive splits of one row block keep the pipeline and the row operand (small n: the operands
  // are L2-resident anyway).  1: u = sp * nrb + rb, CTA b runs the STRIDED units b, b + G, b + 2 G, ... --
  // at any time all CTAs sweep the SAME j-range (split), each for its own row block, nearly in lock
  // step, so a j-tile is fetched from HBM once per time slot instead of once per CTA (n = 2^20: the
  // operands are 630 MB, 5x the L2; contiguous order measured 3.99 TB of DRAM reads per launch at an
  // L2 hit rate of 15%, profiles/r2_mvm_c5_ncu.txt).
  const bool strided = a.unit_order == 1;
  const int u0 = static_cast<int>(blockIdx.x * U / gridDim.x);
  const int u1 = static_cast<int>((blockIdx.x + 1) * U / gridDim.x);
  const int nu = strided ? (U > blockIdx.x ? static_cast<int>((U - 1 - blockIdx.x) / gridDim.x) + 1 : 0) : u1 - u0;
  auto uid = [&](int w) { return strided ? w * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x) : u0 + w; };
  auto u_rb = [&](int u) { return strided ? u % nrb : u / S; };
  auto u_sp = [&](int u) { return strided ? u / nrb : u - (u / S) * S; };
  auto u_jt0 = [&](int u) { return u_sp(u) * per; };
  auto u_nt = [&](int u) { return min(u_jt0(u) + per, ntiles) - u_jt0(u); };
  auto w_newrow = [&](int w) { return w == 0 || u_rb(uid(w)) != u_rb(uid(w - 1)); };
  auto row_barrier = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(THREADS - 64) : "memory"); };  // all but the idle warps
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
    mbar_init(xi_full, 1);
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

  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_ISSUE));
  if (warp == 0) {
    // ---------------- TMA producer (converged warp, elected lane) ----------------
    const uint32_t xjb = static_cast<uint32_t>(BK * a.dp * 4);
    unsigned it = 0;  // unsigned: stage / phase arithmetic without sign fix-ups
    for (int w = 0; w < nu; ++w) {
    const int u = uid(w);
    const int jt0 = u_jt0(u), nt = u_nt(u);
    if (w_newrow(w)) {
      if (w != 0) row_barrier();
      const int row0 = a.row_begin + u_rb(u) * BM;
      if (elect_one()) {
        mbar_arrive_expect_tx(xi_full, BM * a.dp * 4);
        bulk_g2s(sbase + (sXI - base), X32 + static_cast<long long>(row0) * a.dp, BM * a.dp * 4, xi_full);
      }
      __syncwarp();
    }
    for (int lt = 0; lt < nt; ++lt, ++it) {
      const int s = it % SG;
      mbar_wait_sleep(&xv_empty[s], ((it / SG) & 1) ^ 1);
      if (elect_one()) {
        const long long jt = jt0 + lt;
        if constexpr (DIRECT) {
          mbar_arrive_expect_tx(&xv_full[s], 2 * VTILE + xjb);
          bulk_g2s(sbase + (sXJ - base) + s * XJ_TILE, X32 + jt * BK * a.dp, xjb, &xv_full[s]);
        } else {
          mbar_arrive_expect_tx(&xv_full[s], 2 * XG_TILE + BK * 4 + 2 * VTILE + xjb);
          bulk_g2s(sbase + (sXJ - base) + s * XJ_TILE, X32 + jt * BK * a.dp, xjb, &xv_full[s]);
          bulk_g2s(sbase + (sBx - base) + (s * 2 + 0) * XG_TILE, Xh + jt * (BK * 32), XG_TILE, &xv_full[s]);
          bulk_g2s(sbase + (sBx - base) + (s * 2 + 1) * XG_TILE, Xl + jt * (BK * 32), XG_TILE, &xv_full[s]);
          bulk_g2s(sbase + (sN - base) + s * BK * 4, Xn + jt * BK, BK * 4, &xv_full[s]);
        }
        bulk_g2s(sbase + (sV - base) + (s * 2 + 0) * VTILE, Vhi + jt * NPAD * BK, VTILE, &xv_full[s]);
        bulk_g2s(sbase + (sV - base) + (s * 2 + 1) * VTILE, Vlo + jt * NPAD * BK, VTILE, &xv_full[s]);
      }
      __syncwarp();
    }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (converged warp, elected lane) ----------------
    {
      constexpr uint32_t idesc_v = idesc_f16(NPAD);
      constexpr uint32_t idesc_g = tc::idesc_tf32(BK);
      auto gram = [&](unsigned k) {
        if constexpr (DIRECT) return;
        const int s = k % SG, gb = k & 1;
        mbar_wait_sleep(&xv_full[s], (k / SG) & 1);
        mbar_wait_sleep(&g_empty[gb], ((k >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t bh = sBx + (s * 2 + 0) * XG_TILE, bl = sBx + (s * 2 + 1) * XG_TILE;
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const uint32_t ko = ks * 32;  // 8 tf32 along K
            const uint32_t tah = tmem_base + T_AX + ks * 8, tal = tah + 32;
            const uint64_t dbh = tc::smem_desc_sw128(bh + ko), dbl = tc::smem_desc_sw128(bl + ko);
            const uint32_t dg = tmem_base + T_GRAM + gb * BK;
            mma_ts(dg, tah, dbh, idesc_g, ks > 0 ? 1u : 0u);
            mma_ts(dg, tah, dbl, idesc_g, 1u);
            mma_ts(dg, tal, dbh, idesc_g, 1u);
          }
          tc::tc_commit(&g_full[gb]);
        }
        __syncwarp();
        if (lane == 0) GPK_TRACE(7, k);
      };
      unsigned it = 0, gc = 0, rl = 0;
      for (int w = 0; w < nu; ++w) {
      const int u = uid(w);
      const int nt = u_nt(u);
      if (w_newrow(w)) {
        if (w != 0) row_barrier();
        if constexpr (!DIRECT) mbar_wait_sleep(ax_ready, rl & 1);
        ++rl;
        gram(it);
      }
      const bool next_same_row = w + 1 < nu && !w_newrow(w + 1);
      for (int lt = 0; lt < nt; ++lt, ++it) {
        // the next Gram tile overlaps this tile's kernel-shape evaluation (not across a row change)
        if (lt + 1 < nt || next_same_row) gram(it + 1);
        const int s = it % SG, as = it % AS;
        const int buf = gc & 1;
        if (lt % F == 0) mbar_wait_sleep(&acc_empty[buf], ((gc >> 1) & 1) ^ 1);
        mbar_wait_sleep(&a_full[as], (it / AS) & 1);
        if (lane == 0) GPK_TRACE(3, it);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + T_ACC + buf * NPAD;
        const uint32_t tah = tmem_base + T_AT + as * 64, tal = tah + 32;
        const uint32_t bhi = sV + (s * 2 + 0) * VTILE, blo = sV + (s * 2 + 1) * VTILE;
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) {
            const uint32_t koff = ks * 32;  // 16 fp16 along K
            const uint64_t dbh = tc::smem_desc_sw128(bhi + koff), dbl = tc::smem_desc_sw128(blo + koff);
            const uint32_t acc = (lt % F != 0 || ks > 0) ? 1u : 0u;
            mma_ts_f16(d_tmem, tah + ks * 8, dbh, idesc_v, acc);
            mma_ts_f16(d_tmem, tah + ks * 8, dbl, idesc_v, 1u);
            mma_ts_f16(d_tmem, tal + ks * 8, dbh, idesc_v, 1u);
          }
          tc::tc_commit(&a_empty[as]);
          tc::tc_commit(&xv_empty[s]);  // also covers the Gram MMA of this stage and the producers' norm reads
          if (lt % F == F - 1 || lt == nt - 1) tc::tc_commit(&acc_full[buf]);
        }
        __syncwarp();
        if (lt % F == F - 1 || lt == nt - 1) ++gc;
        if (lane == 0) GPK_TRACE(6, it);
      }
      }
    }
  }
  } else {
    // ---------------- producer / epilogue warps ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_PROD));
    const int pw = warp - 4;
    const int lg = warp & 3;   // TMEM lane group
    const int q = pw >> 2;     // 16-column slice of the j-tile, and column-chunk subset of the drain
    const int r = lg * 32 + lane;
    const uint32_t tlane = static_cast<uint32_t>(lg * 32) << 16;
    // (every NC8: 112 registers hold 24 fp32 + 24 fp64 sums without spilling)
    // fp32 TMEM groups are summed in fp32 registers (round to nearest) kConv at a time before the
    // fp64 add: the F2F.F64.F32 conversions share the XU pipe with the MUFUs of the entries
    constexpr bool TWO_LEVEL = true;
    double acc64[HC * 8];
    float acc32[TWO_LEVEL ? HC * 8 : 1];
    int n32 = 0;
#pragma unroll
    for (int e = 0; e < HC * 8; ++e) acc64[e] = 0.0;
    if constexpr (TWO_LEVEL) {
#pragma unroll
      for (int e = 0; e < HC * 8; ++e) acc32[e] = 0.0f;
    }
    float xi[DIRECT ? DPD : 1];
    unsigned it = 0, gce = 0, rl = 0;
    int row = 0;
    float ni = 0.0f;
    for (int w = 0; w < nu; ++w) {
    const int u = uid(w);
    const int jt0 = u_jt0(u), nt = u_nt(u);
    if (w_newrow(w)) {
    if (w != 0) row_barrier();
    row = a.row_begin + u_rb(u) * BM + r;
    ni = DIRECT ? 0.0f : Xn[row];
    if constexpr (!DIRECT) {  // this row's centred coordinates (tf32 hi / lo, columns q*8 .. q*8+7) -> A_x in TMEM
      const long long rb = static_cast<long long>(row >> 3) * 256 + (row & 7) * 32;
      uint32_t h8[8], l8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = q * 8 + u;
        const long long off = rb + ((((k >> 2) ^ (row & 7))) << 2) + (k & 3);
        h8[u] = __float_as_uint(XAh[off]);
        l8[u] = __float_as_uint(XAl[off]);
      }
      tmem_st8(tmem_base + tlane + T_AX + q * 8, h8);
      tmem_st8(tmem_base + tlane + T_AX + 32 + q * 8, l8);
      tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(ax_ready);
    }
    mbar_wait_sleep(xi_full, rl & 1);  // the CTA's fp32 rows (guard path / direct mode)
    ++rl;
    if constexpr (DIRECT) {
#pragma unroll
      for (int k4 = 0; k4 < DPD / 4; ++k4) {
        const float4 v = reinterpret_cast<const float4*>(XIs + r * DPD)[k4];
        xi[4 * k4] = v.x;
        xi[4 * k4 + 1] = v.y;
        xi[4 * k4 + 2] = v.z;
        xi[4 * k4 + 3] = v.w;
      }
    }
    }  // new row block
    auto flush32 = [&]() {
      if constexpr (TWO_LEVEL) {
#pragma unroll
        for (int e = 0; e < HC * 8; ++e) {
          acc64[e] += static_cast<double>(acc32[e]);
          acc32[e] = 0.0f;
        }
        n32 = 0;
      }
    };
    auto drain = [&](unsigned g) {
      const int buf = g & 1;
      mbar_wait_sleep(&acc_full[buf], (g >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int h = 0; h < HC; ++h) {
        const int c8 = q + h * RPT;
        if (c8 < NC8) {
          uint32_t v[8];
          tc::tmem_ld8(tmem_base + tlane + T_ACC + buf * NPAD + c8 * 8, v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if constexpr (TWO_LEVEL) acc32[h * 8 + e] += __uint_as_float(v[e]);
            else acc64[h * 8 + e] += static_cast<double>(__uint_as_float(v[e]));
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[buf]);
      if constexpr (TWO_LEVEL) {
        if (++n32 == kConv) flush32();
      }
    };
    for (int lt = 0; lt < nt; ++lt, ++it) {
      const int s = it % SG, as = it % AS, gb = it & 1;
      if (threadIdx.x == 128) GPK_TRACE(1, it);
      if constexpr (!DIRECT) mbar_wait_sleep(&g_full[gb], (it >> 1) & 1);
      if (threadIdx.x == 128) GPK_TRACE(2, it);
      tc::tc_fence_after();
      // direct mode reads the staged rows; Gram mode reads shared memory only in the (rare)
      // guard path and waits there (the stage is complete: its Gram MMA consumed it)
      if constexpr (DIRECT) mbar_wait_sleep(&xv_full[s], (it / SG) & 1);
      mbar_wait_sleep(&a_empty[as], ((it / AS) & 1) ^ 1);
      // guard threshold of this tile: kGuard (|x_i|^2 + max_j |x_j|^2) bounds every pair's own
      // kGuard (|x_i|^2 + |x_j|^2), so a warp whose 8 entries all exceed it has no near pair
#ifdef GPK_TCG_EXACT_GUARD  // experiment: every group takes the exact per-entry test
      const float gthr = 3.0e38f;
#else
      const float gthr = DIRECT ? 0.0f : kGuard * (ni + __ldg(Xtm + jt0 + lt));
#endif
      // the thread's 16 Gram values in one TMEM load and the Gram buffer released right away
      // (measured: -2% at NC8 = 7; with NC8 > 8 the extra live registers cost 6%, so there the
      // two halves load separately)
      constexpr bool G16 = !DIRECT;  // (with 112 registers per producer thread the single load also pays for NC8 > 8)
      uint32_t gv16[G16 ? 16 : 8];
      if constexpr (G16) {
        tmem_ld16(tmem_base + tlane + T_GRAM + gb * BK + q * JPT, gv16);
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&g_empty[gb]);
      }
      if (threadIdx.x == 128) GPK_TRACE(5, it);
#pragma unroll
      for (int hf8 = 0; hf8 < 2; ++hf8) {  // two halves of 8 entries: Gram -> s -> entry -> TMEM
        float sv[8];
        if constexpr (DIRECT) {  // fp32 direct differences, two entries per paired FFMA2
          const float* xjb = XJs + s * (XJ_TILE / 4) + (q * JPT + hf8 * 8) * DPD;
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            float2 acc2 = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int k4 = 0; k4 < DPD / 4; ++k4) {
              const float4 a4 = reinterpret_cast<const float4*>(xjb + u * DPD)[k4];
              const float4 b4 = reinterpret_cast<const float4*>(xjb + (u + 1) * DPD)[k4];
              const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 df = __ffma2_rn(make_float2(av[e], bv[e]), make_float2(1.0f, 1.0f),
                                             make_float2(-xi[4 * k4 + e], -xi[4 * k4 + e]));
                acc2 = __ffma2_rn(df, df, acc2);
              }
            }
            sv[u] = acc2.x;
            sv[u + 1] = acc2.y;
          }
        } else {
        const uint32_t* gv = gv16 + (G16 ? hf8 * 8 : 0);
        if constexpr (!G16) {
          tc::tmem_ld8(tmem_base + tlane + T_GRAM + gb * BK + q * JPT + hf8 * 8, gv16);
          tc::tmem_wait_ld();
          if (hf8 == 1) {
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&g_empty[gb]);
          }
        }
        // s_ij straight from the augmented Gram MMA (n_i + n_j - 2 x~_i . x~_j)
#pragma unroll
        for (int u = 0; u < 8; ++u) sv[u] = __uint_as_float(gv[u]);
        const float smin = fminf(fminf(fminf(sv[0], sv[1]), fminf(sv[2], sv[3])),
                                 fminf(fminf(sv[4], sv[5]), fminf(sv[6], sv[7])));
        // Cancellation guard: s <= kGuard (|x_i|^2 + |x_j|^2) (near pairs, incl. the diagonal,
        // where the expanded form may even go negative) is recomputed from fp32 direct
        // differences of the un-centred coordinates, so the expanded form only serves pairs whose
        // relative error in s stays at the fp32 level.  Every entry that is not a near pair
        // exceeds kGuard (|x_i|^2 + |x_j|^2) >= 0, hence is positive: no clamp anywhere.
        if (__any_sync(0xffffffffu, smin <= gthr)) {
          // some entry is within the tile bound: the exact per-entry test first (cheap), the
          // direct recompute only when an entry really is a near pair
          mbar_wait_sleep(&xv_full[s], (it / SG) & 1);  // the stage's norms and rows, generic proxy
          const float* nsj = Ns + s * BK + q * JPT + hf8 * 8;
          const float4 n0 = reinterpret_cast<const float4*>(nsj)[0], n1 = reinterpret_cast<const float4*>(nsj)[1];
          const float nj[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
          bool near[8];
          bool anyn = false;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            near[u] = sv[u] <= kGuard * (nj[u] + ni);
            anyn = anyn || near[u];
          }
          // Low-dimensional data (d + 2 <= 16: KS <= 2) with short lengthscales have near pairs on a
          // large share of their tiles (C3: the tile bound fires on half of the 8-entry groups, a real
          // near pair sits in a quarter of them): there only the lanes that hold a near pair recompute
          // it (typically one lane, one entry) -- C3 1.74 -> 1.48 ms, C5 974 -> 936 ms per launch.  In
          // higher dimension near pairs are the diagonal tile's business and the whole warp walks the 8
          // entries together (no divergence, the schedule C2 was tuned with).
          constexpr bool DIVG = KS <= 2;
          if constexpr (DIVG) {
            if (anyn) {
              const float4* xi4 = reinterpret_cast<const float4*>(XIs + r * a.dp);
              const float4* xj4 =
                  reinterpret_cast<const float4*>(XJs + s * (XJ_TILE / 4) + (q * JPT + hf8 * 8) * a.dp);
              const int d4 = a.dp >> 2;
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                if (near[u]) {
                  float acc = 0.0f;
#pragma unroll 1
                  for (int k = 0; k < d4; ++k) {
                    const float4 p = xi4[k], qv = xj4[u * d4 + k];
                    const float d0 = p.x - qv.x, d1 = p.y - qv.y, d2 = p.z - qv.z, d3 = p.w - qv.w;
                    acc = fmaf(d0, d0, acc);
                    acc = fmaf(d1, d1, acc);
                    acc = fmaf(d2, d2, acc);
                    acc = fmaf(d3, d3, acc);
                  }
                  sv[u] = acc;
                }
              }
            }
            __syncwarp();
          } else if (__any_sync(0xffffffffu, anyn)) {
            // the whole warp evaluates the 8 direct distances (no divergence), from shared memory
            const float4* xi4 = reinterpret_cast<const float4*>(XIs + r * a.dp);
            const float4* xj4 =
                reinterpret_cast<const float4*>(XJs + s * (XJ_TILE / 4) + (q * JPT + hf8 * 8) * a.dp);
            const int d4 = a.dp >> 2;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              float acc = 0.0f;
#pragma unroll 1
              for (int k = 0; k < d4; ++k) {
                const float4 p = xi4[k], qv = xj4[u * d4 + k];
                const float d0 = p.x - qv.x, d1 = p.y - qv.y, d2 = p.z - qv.z, d3 = p.w - qv.w;
                acc = fmaf(d0, d0, acc);
                acc = fmaf(d1, d1, acc);
                acc = fmaf(d2, d2, acc);
                acc = fmaf(d3, d3, acc);
              }
              if (near[u]) sv[u] = acc;
            }
          }
        }
        }  // Gram mode
        uint32_t eh[4], el[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const float2 e2 = kval32x2_scaled<FAM, kEntryLog2>(make_float2(sv[2 * p], sv[2 * p + 1]));
          eh[p] = split_f16x2(e2, el[p]);
        }
        tmem_st4(tmem_base + tlane + T_AT + as * 64 + q * 8 + hf8 * 4, eh);
        tmem_st4(tmem_base + tlane + T_AT + as * 64 + 32 + q * 8 + hf8 * 4, el);
      }
      tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&a_full[as]);
      if (lane == 0 && it < 64) GPK_TRACE(4, it * 16 + pw);
      if (lt % F == 0 && lt > 0) drain(gce++);
    }
    drain(gce++);
    flush32();
    if (threadIdx.x == 128) GPK_TRACE(0, 2);
    if (row < a.row_end) {
      double* o = out + static_cast<long long>(u_sp(u)) * a.split_stride;
#pragma unroll
      for (int h = 0; h < HC; ++h) {
        const int c8 = q + h * RPT;
        if (c8 >= NC8) continue;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int col = c8 * 8 + e;
          if (col < a.t) o[static_cast<long long>(col) * a.ldo + (row - a.row_begin)] = colscale[col] * acc64[h * 8 + e];
        }
      }
    }
#pragma unroll
    for (int e = 0; e < HC * 8; ++e) acc64[e] = 0.0;
    (void)jt0;
    }  // units
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
  return 1024 + SG * 2 * XG_TILE + SG * 2 * (8 * NC8 * BK * 2) + SG * BK * 4 + SG * XJ_TILE + XI_BLOCK +
         (2 * SG + 2 * AS + 10) * 8 + 16;
}

template <int FAM, int KS, int NC8, int DPD>
cudaError_t launch_tcg_t(const float* Xh, const float* Xl, const float* Xn, const float* X32, const __half* Vhi,
                         const __half* Vlo, const double* colscale, double* out, const MvmArgs& a, dim3 grid,
                         cudaStream_t st) {
  constexpr size_t sm = tcg_smem_bytes<NC8>();
  static_assert(sm <= 232448, "tcg smem");
  auto k = fused_kmvm_tcg_kernel<FAM, KS, NC8, DPD>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k<<<grid, THREADS, sm, st>>>(Xh, Xl, Xn, X32, Vhi, Vlo, colscale, out, a);
  return cudaGetLastError();
}

template <int FAM>
cudaError_t launch_tcg_fam(int ks, int dpd, int nc8, const float* Xh, const float* Xl, const float* Xn,
                           const float* X32, const __half* Vhi, const __half* Vlo, const double* colscale,
                           double* out, const MvmArgs& a, dim3 g, cudaStream_t st) {
#define GPK_TCG_ARGS Xh, Xl, Xn, X32, Vhi, Vlo, colscale, out, a, g, st
  if (dpd > 0) {  // direct-difference mode
#define GPK_TCG_ND(N)                                                \
  case N:                                                            \
    switch (dpd) {                                                   \
      case 4: return launch_tcg_t<FAM, 0, N, 4>(GPK_TCG_ARGS);       \
      case 8: return launch_tcg_t<FAM, 0, N, 8>(GPK_TCG_ARGS);       \
      default: return cudaErrorInvalidValue;                         \
    }
    switch (nc8) {
      GPK_TCG_ND(1) GPK_TCG_ND(2) GPK_TCG_ND(4) GPK_TCG_ND(6) GPK_TCG_ND(7) GPK_TCG_ND(8) GPK_TCG_ND(9)
      GPK_TCG_ND(10) GPK_TCG_ND(12)
      default: break;
    }
#undef GPK_TCG_ND
    return cudaErrorInvalidValue;
  }
  if constexpr (FAM == kMatern12) {
    return cudaErrorInvalidValue;  // Matern-1/2 is never evaluated from expanded distances
  } else {
#define GPK_TCG_NC(N)                                               \
  case N:                                                           \
    switch (ks) {                                                   \
      case 1: return launch_tcg_t<FAM, 1, N, 0>(GPK_TCG_ARGS);      \
      case 2: return launch_tcg_t<FAM, 2, N, 0>(GPK_TCG_ARGS);      \
      case 3: return launch_tcg_t<FAM, 3, N, 0>(GPK_TCG_ARGS);      \
      case 4: return launch_tcg_t<FAM, 4, N, 0>(GPK_TCG_ARGS);      \
      default: return cudaErrorInvalidValue;                        \
    }
    switch (nc8) {
      GPK_TCG_NC(1) GPK_TCG_NC(2) GPK_TCG_NC(4) GPK_TCG_NC(6) GPK_TCG_NC(7) GPK_TCG_NC(8) GPK_TCG_NC(9)
      GPK_TCG_NC(10) GPK_TCG_NC(12)
      default: break;
    }
#undef GPK_TCG_NC
    return cudaErrorInvalidValue;
  }
#undef GPK_TCG_ARGS
}

}  // namespace tcg
}  // namespace gpk

#define GPK_INSTANTIATE_TCG_FAMILY(FAM)                                                                      \
  namespace gpk {                                                                                            \
  namespace tcg {                                                                                            \
  template cudaError_t launch_tcg_fam<FAM>(int, int, int, const float*, const float*, const float*, const float*, \
                                           const __half*, const __half*, const double*, double*,             \
                                           const MvmArgs&, dim3, cudaStream_t);                              \
  }                                                                                                          \
  }
