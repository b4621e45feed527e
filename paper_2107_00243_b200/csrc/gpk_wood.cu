// Shared-memory-staged Woodbury GEMMs for the fused single-rank CG iteration
// (preconditioners.hpp:114-118, DiagPlusLowRank::solve_matrix):
//
//   G1s: W = L^T r_new              (k x t, reduction over the n rows)
//        fused with x += alpha p, r -= alpha (Kp + s2 p)            (krylov.hpp:94-95)
//   G2s: z = (r - C W) / s2 and per-CTA r.z / z.z partials
//   cg_beta_p: beta from those partials + p = z + beta p             (krylov.hpp:96-119)
//
// Both kernels give every CTA one contiguous run of rows (16-row units, the partition
// is a function of n and the grid only), stage 64x64 fp64 operand tiles in padded shared
// memory (stride 68 doubles: every m8n8k4 fragment load is bank-conflict free) and run the
// products on the fp64 tensor cores (DMMA 8x8x4).  Warp w owns output m-tile w of the
// 64x64 tile and walks K in fixed order, so every output element is a fixed-order sum of
// its own row and column only (the batched == independent contract of krylov.hpp:131-132)
// and reruns are bitwise reproducible.  The earlier g1/g2 kernels (gpk_linalg.cu,
// gpk_cgfused.cu) read fragments straight from global memory (each m-tile warp re-read the
// R block) and were latency bound: 23 / 45 us per launch at C2 (profiles/r1_wood_*).
#include <algorithm>
#include <cstdlib>
#include <cfloat>
#include <cstdint>

#include <cooperative_groups.h>

#include "gpk_common.cuh"
#include "gpk_linalg.h"

namespace gpk {

namespace {

constexpr int kWT = 256;   // threads per CTA (8 warps)
constexpr int kWS = 64;    // tile edge: rows per sub-chunk, columns per group, K per slab
constexpr int kSR = 72;    // smem row stride (doubles) of the K-permuted tiles; 36 = 4 (mod 8) units
constexpr int kUnit = 16;  // row-partition granularity
constexpr size_t kWSmem = 2ull * kWS * kSR * sizeof(double);  // 73728 B: two tiles

// K permutation inside a 64-long K tile: DMMA k-step q (0..15) takes K indices
// {q, 16 + q, 32 + q, 48 + q}, lane r the index 16 r + q, stored at r * 18 + q.  A lane's
// operands of k-steps q and q + 1 are adjacent (one LDS.128 for two DMMAs) and the 8 lanes
// of a 128-bit phase hit distinct bank groups (row stride 72 doubles).  The sum over K is
// the same set of products in a fixed, different order (deterministic).
GPK_DEV int kpos(int kidx) { return (kidx >> 4) * 18 + (kidx & 15); }

GPK_DEV void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// asynchronous copy of the element pair src[0..1] -> dst[0..1] (nv valid elements, the rest
// zero-filled): one 16-byte cp.async when VEC (16-byte aligned source), else two 8-byte ones
template <bool VEC>
GPK_DEV void cp_pair(double* dst, const double* src, int nv, const double* safe) {
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
GPK_DEV void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// rows [r0, r1) of CTA b out of G: contiguous runs of 16-row units
GPK_DEV void rows_of(int b, int G, int n, int& r0, int& r1) {
  const long long nu = (n + kUnit - 1) / kUnit;
  r0 = static_cast<int>(nu * b / G) * kUnit;
  r1 = min(n, static_cast<int>(nu * (b + 1) / G) * kUnit);
}

int sm_count() {
  static int c = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return c;
}

}  // namespace

// ---- G1s: part[b][s][kk] = sum over CTA b's rows i of A[kk][i] * Rn[s][i]
// XR: Rn = R - alpha_s (Y + s2 P) for live slots, written back to R (and X += alpha P) by
// the CTA that owns the rows (no other CTA reads them).  NT = 8-column tiles of the group.
// Copy thread map: pair p = tid & 31 (elements 2p, 2p+1 of a 64-long row), rows tid / 32 + 8e.
// One 64-column group [s0, s0 + ns) of CTA b out of G (the body of g1s_kernel, also run as a
// phase of the cooperative CG iteration, gpk_cgcoop.cu).  The slot states are read through
// L2 (they may have been written earlier in the same cooperative launch).
template <bool XR, bool VEC, int NT>
GPK_DEV void g1s_group(int b, int G, int s0, const double* __restrict__ A, long long lda, int ka,
                       double* __restrict__ R, long long ldr, int tb, int n, double* __restrict__ part,
                       double* __restrict__ X, const double* __restrict__ P, const double* __restrict__ Y, double sig2,
                       const SlotState* ss, double* wsm, double* s_al) {
  double* As = wsm;              // [kk][kpos(i)]
  double* Bs = wsm + kWS * kSR;  // [s][kpos(i)]
  int r0, r1;
  rows_of(b, G, n, r0, r1);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, r = lane & 3, m = lane >> 2;
  const int cp = tid & 31, crow = tid >> 5, cpos = kpos(2 * cp);
  const int ns = min(kWS, tb - s0);
  if (XR) {
    if (tid < ns) {
      const SlotState* x = ss + s0 + tid;
      s_al[tid] = __ldcg(&x->flag) == 0 ? __ldcg(&x->alpha) : 0.0;
    }
  }
  for (int k0 = 0; k0 < ka; k0 += kWS) {
    const int nk = min(kWS, ka - k0), mtc = (nk + 7) >> 3;
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
    for (int i0 = r0; i0 < r1; i0 += kWS) {
      const int ni = min(kWS, r1 - i0);
      const int nv = min(2, max(0, ni - 2 * cp));  // valid elements of this thread's pair
      __syncthreads();  // the previous tile's fragments are consumed
#pragma unroll
      for (int e = 0; e < kWS / 8; ++e) {  // A tile rows kk (garbage rows >= nk feed unwritten outputs)
        const int kk = crow + 8 * e;
        if (kk < mtc * 8)
          cp_pair<VEC>(As + kk * kSR + cpos, A + (k0 + min(kk, nk - 1)) * lda + i0 + 2 * cp, nv, A);
      }
      if (!XR || k0 > 0) {
#pragma unroll
        for (int e = 0; e < kWS / 8; ++e) {
          const int s = crow + 8 * e;
          if (s < NT * 8) cp_pair<VEC>(Bs + s * kSR + cpos, R + (s0 + min(s, ns - 1)) * ldr + i0 + 2 * cp, nv, R);
        }
      } else {
        // x += alpha p, r -= alpha (Kp + s2 p) (krylov.hpp:94-95, cg_update_xr_kernel's
        // expressions): all loads of 2 rows in flight, then the updates
#pragma unroll
        for (int e0 = 0; e0 < kWS / 8; e0 += 2) {
          double rv[2][2], pv[2][2], yv[2][2], xv[2][2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int s = crow + 8 * (e0 + u);
            const bool v = s < ns;
            const long long o = (s0 + (v ? s : 0)) * ldr + i0 + 2 * cp;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const bool vh = v && h < nv;
              rv[u][h] = vh ? R[o + h] : 0.0;
              pv[u][h] = vh ? P[o + h] : 0.0;
              yv[u][h] = vh ? Y[o + h] : 0.0;
              xv[u][h] = vh ? X[o + h] : 0.0;
            }
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int s = crow + 8 * (e0 + u);
            if (s >= NT * 8) continue;
            const bool v = s < ns;
            const double a = v ? s_al[s] : 0.0;
            const long long o = (s0 + (v ? s : 0)) * ldr + i0 + 2 * cp;
            double2 out;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              double r2 = rv[u][h];
              if (a != 0.0 && h < nv) {  // live slot (alpha > 0 is checked by alpha_step)
                const double ap = yv[u][h] + sig2 * pv[u][h];
                X[o + h] = xv[u][h] + a * pv[u][h];
                r2 -= a * ap;
                R[o + h] = r2;
              }
              (h ? out.y : out.x) = r2;
            }
            *reinterpret_cast<double2*>(Bs + s * kSR + cpos) = out;
          }
        }
      }
      cp_wait_all();
      __syncthreads();
      if (w < mtc) {
        const double* ap = As + (w * 8 + m) * kSR + r * 18;
        const double* bp = Bs + m * kSR + r * 18;
#pragma unroll 2
        for (int q = 0; q < 16; q += 2) {
          const double2 a = *reinterpret_cast<const double2*>(ap + q);
          double2 bb[NT];
#pragma unroll
          for (int j = 0; j < NT; ++j) bb[j] = *reinterpret_cast<const double2*>(bp + j * 8 * kSR + q);
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[j], a.x, bb[j].x);  // independent accumulators first
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[j], a.y, bb[j].y);
        }
      }
    }
    if (w < mtc) {
      const int kk = k0 + w * 8 + m;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int s = s0 + 8 * j + 2 * r + e;
          if (s < tb && kk < ka) part[(static_cast<long long>(b) * tb + s) * ka + kk] = acc[j][e];
        }
    }
  }
}

template <bool XR, bool VEC, int NT>
__global__ void __launch_bounds__(kWT, 2)
    g1s_kernel(const double* __restrict__ A, long long lda, int ka, double* __restrict__ R, long long ldr, int tb,
               int s_off, int n, double* __restrict__ part, double* __restrict__ X, const double* __restrict__ P,
               const double* __restrict__ Y, double sig2, const SlotState* __restrict__ ss) {
  extern __shared__ __align__(16) double wsm[];
  __shared__ double s_al[kWS];  // alpha of live slots, 0 for frozen ones (XR)
  g1s_group<XR, VEC, NT>(blockIdx.x, gridDim.x, s_off + blockIdx.y * kWS, A, lda, ka, R, ldr, tb, n, part, X, P, Y,
                         sig2, ss, wsm, s_al);
}

// W[s][kk] = sum over the G CTA partials in fixed order.  A CTA owns 32 consecutive outputs
// (coalesced 256-byte rows of the partial array); warp q sums partials q, q + 8, ... (16
// loads in flight per thread), and the 8 warp sums are combined in warp order.
GPK_DEV void g1s_reduce_chunk(long long chunk, const double* part, int G, int ka, int tb, double* W, long long ldw,
                              double (*red)[32]) {
  const int o = threadIdx.x & 31, q = threadIdx.x >> 5;
  const long long idx = chunk * 32 + o;
  const long long tot = static_cast<long long>(ka) * tb;
  double acc = 0.0;
  if (idx < tot) {
    const double* p = part + idx;
    int c = q;
    for (; c + 8 * 15 < G; c += 8 * 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcg(p + static_cast<long long>(c + 8 * u) * tot);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc += v[u];
    }
    for (; c < G; c += 8) acc += __ldcg(p + static_cast<long long>(c) * tot);
  }
  red[q][o] = acc;
  __syncthreads();
  if (q == 0 && idx < tot) {
    double sum = red[0][o];
#pragma unroll
    for (int u = 1; u < 8; ++u) sum += red[u][o];
    const int s = static_cast<int>(idx / ka), kk = static_cast<int>(idx % ka);
    W[s * ldw + kk] = sum;
  }
}

__global__ void __launch_bounds__(256) g1s_reduce_kernel(const double* __restrict__ part, int G, int ka, int tb,
                                                         double* __restrict__ W, long long ldw) {
  __shared__ double red[8][32];
  g1s_reduce_chunk(blockIdx.x, part, G, ka, tb, W, ldw, red);
}

// ---- G2s: Z = R / s2 - (C W) / s2 on CTA b's rows, per-CTA r.z / z.z partials, then a
// two-level last-arrival reduction (groups of 32 CTAs, then the groups) runs beta_step.
GPK_DEV void beta_step_s(SlotState& x, double rz_new, double zz, int k, double rel_tol, double* beta_hist,
                         double* resid_hist, int max_iters) {
  if (x.flag != 0) {
    x.beta = 0.0;
    return;
  }
  if (!isfinite(rz_new) || rz_new < 0.0) {
    x.status = kStatusRz;
    x.bad = rz_new;
    x.iters = k;
    x.flag = kFlagError;
    x.beta = 0.0;
    return;
  }
  const double pres = sqrt(zz);
  const long long base = static_cast<long long>(x.col) * max_iters + (k - 1);
  if (resid_hist) resid_hist[base] = pres;
  x.iters = k;
  x.pres = pres;
  if (pres <= rel_tol * x.norm0 || rz_new == 0.0) {
    x.flag = kFlagConverged;
    x.beta = 0.0;
    return;
  }
  const double beta = rz_new / x.rz;
  if (beta_hist) beta_hist[base] = beta;
  x.beta = beta;
  x.rz = rz_new;
}

// ---- beta + p update (krylov.hpp:96-119): every CTA of column s sums the G2s partials in
// the same fixed order (identical rz_new, zz), runs beta_step on its own copy of the slot
// state and updates its rows of p = z + beta p with the |p| maxima of the next fp16 pack;
// the LAST CTA of the column to arrive (every other one has read the old state by then)
// stores the updated state.  This replaces G2s's last-arrival tail, during which the rest
// of the GPU idled (ncu: SMs active 56% of the G2s elapsed time).
__global__ void __launch_bounds__(kWT) cg_beta_p_kernel(double* __restrict__ P, const double* __restrict__ Z, int n,
                                                        long long ldn, SlotState* __restrict__ ss,
                                                        const double* __restrict__ prz,
                                                        const double* __restrict__ pzz, int G,
                                                        unsigned* __restrict__ cnt, int k, double rel_tol,
                                                        double* __restrict__ beta_hist,
                                                        double* __restrict__ resid_hist, int max_iters,
                                                        unsigned long long* __restrict__ vmax,
                                                        SlotState* __restrict__ snap) {
  __shared__ double red[kWT / 32];
  const int s = blockIdx.y, tid = threadIdx.x;
  SlotState x = ss[s];
  double a = 0.0, z = 0.0;
  for (int b = tid; b < G; b += kWT) {  // thread-strided, then the fixed block tree
    a += __ldcg(prz + static_cast<long long>(s) * G + b);
    z += __ldcg(pzz + static_cast<long long>(s) * G + b);
  }
  const double rz_new = block_sum(a, red);
  const double zz = block_sum(z, red);
  const bool first = blockIdx.x == 0;
  beta_step_s(x, rz_new, zz, k, rel_tol, first ? beta_hist : nullptr, first ? resid_hist : nullptr, max_iters);
  const bool live = x.flag == 0;
  const double beta = x.beta;
  double mx = 0.0;
  for (int i = blockIdx.x * kWT + tid; i < n; i += gridDim.x * kWT) {
    const long long o = s * ldn + i;
    double p = P[o];
    if (live) {
      p = Z[o] + beta * p;  // krylov.hpp:116 (cg_update_p_kernel's expression)
      P[o] = p;
    }
    mx = fmax(mx, fabs(p));
  }
  if (vmax) {  // CTA maximum first: one atomic per CTA (order-independent, so deterministic)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < kWT / 32; ++q) mx = fmax(mx, red[q]);
      if (mx > 0.0) atomicMax(vmax + s, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(cnt + s, 1u) == gridDim.x - 1) {
      ss[s] = x;
      cnt[s] = 0;
      // the host's copy of the slot state, straight into pinned memory (the host reads it after
      // an event recorded behind this kernel: no system-scope fence needed here; one cost ~3 us)
      if (snap) snap[s] = x;
    }
  }
}

// Z tile operand layout: Cs[kk][i ^ 4 ((kk >> 4) & 3)] (row stride 64): the A fragments of
// the permuted k-steps are conflict-free 64-bit loads; pairs (2p, 2p+1) stay adjacent.
GPK_DEV int cswz(int kk) { return ((kk >> 4) & 3) * 4; }

// One column group [s0, s0 + ns) of G2s (the launcher runs one launch per group; group
// launches use disjoint counters and partial columns).
template <bool VEC, int NT>
GPK_DEV void g2s_group(int b, int G, const double* __restrict__ C, long long ldc, int ka, const double* W,
                       long long ldw, int s0, int ns, int n, double* __restrict__ Z, const double* R, long long ldn,
                       double sig2, double* __restrict__ prz, double* __restrict__ pzz, double* wsm,
                       double (*srz)[kWS], double (*szz)[kWS]) {
  double* Cs = wsm;              // [kk][i ^ cswz(kk)], stride 64
  double* Ws = wsm + kWS * kSR;  // [s][kpos(kk)], stride 72
  int r0, r1;
  rows_of(b, G, n, r0, r1);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, r = lane & 3, m = lane >> 2;
  const int cp = tid & 31, crow = tid >> 5;
  double crun = 0.0, zrun = 0.0;  // thread c < 64: the CTA's running sums of column s0 + c
  for (int i0 = r0; i0 < r1; i0 += kWS) {
    const int ni = min(kWS, r1 - i0), mtc = (ni + 7) >> 3;
    const int nvi = min(2, max(0, ni - 2 * cp));
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
    for (int k0 = 0; k0 < ka; k0 += kWS) {
      const int nk = min(kWS, ka - k0);
      const int nvk = min(2, max(0, nk - 2 * cp));
      __syncthreads();
#pragma unroll
      for (int e = 0; e < kWS / 8; ++e) {  // Cs rows kk >= nk are zero (K dimension)
        const int kk = crow + 8 * e;
        cp_pair<VEC>(Cs + kk * kWS + ((2 * cp) ^ cswz(kk)), C + (k0 + min(kk, nk - 1)) * ldc + i0 + 2 * cp,
                     kk < nk ? nvi : 0, C);
      }
#pragma unroll
      for (int e = 0; e < kWS / 8; ++e) {  // Ws[s][kpos(kk)] = W[s0 + s][k0 + kk], zero for kk >= nk
        const int sl = crow + 8 * e;
        if (sl < NT * 8)
          cp_pair<VEC>(Ws + sl * kSR + kpos(2 * cp), W + (s0 + min(sl, ns - 1)) * ldw + k0 + 2 * cp, nvk, W);
      }
      cp_wait_all();
      __syncthreads();
      if (w < mtc) {
        const double* ap = Cs + r * 16 * kWS + ((w * 8 + m) ^ (4 * r));
        const double* bp = Ws + m * kSR + r * 18;
#pragma unroll 2
        for (int q = 0; q < 16; q += 2) {
          const double a0 = ap[q * kWS], a1 = ap[(q + 1) * kWS];
          double2 bb[NT];
#pragma unroll
          for (int j = 0; j < NT; ++j) bb[j] = *reinterpret_cast<const double2*>(bp + j * 8 * kSR + q);
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[j], a0, bb[j].x);  // independent accumulators first
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[j], a1, bb[j].y);
        }
      }
    }
    // z and the lane's r.z / z.z contributions (row i0 + 8w + m, columns s0 + 8j + 2r + e)
    const int row = i0 + w * 8 + m;
    const bool rowv = w < mtc && row < r1;
    double crz[NT][2], czz[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {  // all loads first
        const int sl = 8 * j + 2 * r + e;
        crz[j][e] = (rowv && sl < ns) ? R[static_cast<long long>(s0 + sl) * ldn + row] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int sl = 8 * j + 2 * r + e;
        const double rr = crz[j][e];
        czz[j][e] = 0.0;
        if (rowv && sl < ns) {
          const double z = rr / sig2 - acc[j][e] / sig2;  // preconditioners.hpp:114-118
          Z[static_cast<long long>(s0 + sl) * ldn + row] = z;
          crz[j][e] = rr * z;
          czz[j][e] = z * z;
        }
      }
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          crz[j][e] += __shfl_xor_sync(0xffffffffu, crz[j][e], o);
          czz[j][e] += __shfl_xor_sync(0xffffffffu, czz[j][e], o);
        }
    if (m == 0) {
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          srz[w][8 * j + 2 * r + e] = crz[j][e];
          szz[w][8 * j + 2 * r + e] = czz[j][e];
        }
    }
    __syncthreads();
    if (tid < NT * 8) {
      for (int q = 0; q < 8; ++q) {  // the sub-chunk's rows in warp order
        crun += srz[q][tid];
        zrun += szz[q][tid];
      }
    }
  }
  if (tid < ns) {
    prz[static_cast<long long>(s0 + tid) * G + b] = crun;
    pzz[static_cast<long long>(s0 + tid) * G + b] = zrun;
  }
}

template <bool VEC, int NT>
__global__ void __launch_bounds__(kWT, 2)
    g2s_dots_beta_kernel(const double* __restrict__ C, long long ldc, int ka, const double* __restrict__ W,
                         long long ldw, int s0, int ns, int n, double* __restrict__ Z, const double* __restrict__ R,
                         long long ldn, double sig2, double* __restrict__ prz, double* __restrict__ pzz) {
  extern __shared__ __align__(16) double wsm[];
  __shared__ double srz[8][kWS], szz[8][kWS];
  g2s_group<VEC, NT>(blockIdx.x, gridDim.x, C, ldc, ka, W, ldw, s0, ns, n, Z, R, ldn, sig2, prz, pzz, wsm, srz, szz);
}

int wood_grid() {  // CTAs per SM: 2 (env GPK_WOOD_CPS=1 for A/B checks)
  static int cps = [] {
    const char* e = std::getenv("GPK_WOOD_CPS");
    return e && std::atoi(e) == 1 ? 1 : 2;
  }();
  return cps * sm_count();
}

size_t wood_g1_workspace(int ka, int tb) { return static_cast<size_t>(wood_grid()) * ka * tb; }
// prz, pzz: tb * G each
size_t wood_g2_partials(int tb) { return static_cast<size_t>(tb) * wood_grid(); }

namespace {

template <class K>
cudaError_t set_smem(K kern) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kWSmem));
}

template <bool XR, bool VEC, int NT>
cudaError_t g1s_launch(dim3 g, cudaStream_t st, const double* A, long long lda, int ka, double* R, long long ldr,
                       int tb, int s_off, int n, double* part, double* X, const double* P, const double* Y, double sig2,
                       const SlotState* ss) {
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = set_smem(g1s_kernel<XR, VEC, NT>);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  g1s_kernel<XR, VEC, NT><<<g, kWT, kWSmem, st>>>(A, lda, ka, R, ldr, tb, s_off, n, part, X, P, Y, sig2, ss);
  return cudaGetLastError();
}

template <bool XR, bool VEC>
cudaError_t g1s_dispatch(int nt, dim3 g, cudaStream_t st, const double* A, long long lda, int ka, double* R,
                         long long ldr, int tb, int s_off, int n, double* part, double* X, const double* P,
                         const double* Y, double sig2, const SlotState* ss) {
#define GPK_G1S(NTV) \
  case NTV:          \
    return g1s_launch<XR, VEC, NTV>(g, st, A, lda, ka, R, ldr, tb, s_off, n, part, X, P, Y, sig2, ss);
  switch (nt) {
    GPK_G1S(1) GPK_G1S(2) GPK_G1S(3) GPK_G1S(4) GPK_G1S(5) GPK_G1S(6) GPK_G1S(7) GPK_G1S(8)
  }
#undef GPK_G1S
  return cudaErrorInvalidValue;
}

template <bool VEC, int NT>
cudaError_t g2s_launch(cudaStream_t st, const double* C, long long ldc, int ka, const double* W, long long ldw,
                       int s0, int ns, int n, double* Z, const double* R, long long ldn, double sig2, double* prz,
                       double* pzz) {
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = set_smem(g2s_dots_beta_kernel<VEC, NT>);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  g2s_dots_beta_kernel<VEC, NT><<<wood_grid(), kWT, kWSmem, st>>>(C, ldc, ka, W, ldw, s0, ns, n, Z, R, ldn, sig2,
                                                                   prz, pzz);
  return cudaGetLastError();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

cudaError_t launch_g1s(const double* A, long long lda, int ka, double* R, long long ldr, int tb, int n,
                       double* part, double* W, long long ldw, double* X, const double* P, const double* Y,
                       double sig2, const SlotState* ss, cudaStream_t st) {
  if (ka <= 0 || tb <= 0) return cudaSuccess;
  const int G = wood_grid();
  const bool vec = aligned16(A) && aligned16(R) && lda % 2 == 0 && ldr % 2 == 0;
  cudaError_t e = cudaSuccess;
  const int full = tb / kWS, rem = tb % kWS;
  for (int grp = 0; grp < 2 && e == cudaSuccess; ++grp) {  // full 64-column groups, then the rest
    const int ngy = grp == 0 ? full : (rem ? 1 : 0);
    if (ngy == 0) continue;
    const int nt = grp == 0 ? 8 : (rem + 7) / 8, s_off = grp == 0 ? 0 : full * kWS;
    const dim3 g(G, ngy);
    if (X)
      e = vec ? g1s_dispatch<true, true>(nt, g, st, A, lda, ka, R, ldr, tb, s_off, n, part, X, P, Y, sig2, ss)
              : g1s_dispatch<true, false>(nt, g, st, A, lda, ka, R, ldr, tb, s_off, n, part, X, P, Y, sig2, ss);
    else
      e = vec ? g1s_dispatch<false, true>(nt, g, st, A, lda, ka, R, ldr, tb, s_off, n, part, nullptr, nullptr,
                                          nullptr, 0.0, nullptr)
              : g1s_dispatch<false, false>(nt, g, st, A, lda, ka, R, ldr, tb, s_off, n, part, nullptr, nullptr,
                                           nullptr, 0.0, nullptr);
  }
  if (e != cudaSuccess) return e;
  const long long tot = static_cast<long long>(ka) * tb;
  g1s_reduce_kernel<<<static_cast<unsigned>((tot + 31) / 32), 256, 0, st>>>(part, G, ka, tb, W, ldw);
  return cudaGetLastError();
}

cudaError_t launch_g2s_dots_beta(const double* C, long long ldc, int ka, const double* W, long long ldw, int tb,
                                 int n, double* Z, const double* R, long long ldn, double sig2, double* prz,
                                 double* pzz, cudaStream_t st) {
  if (tb <= 0) return cudaSuccess;
  const bool vec = aligned16(C) && aligned16(W) && ldc % 2 == 0 && ldw % 2 == 0;
  for (int s0 = 0; s0 < tb; s0 += kWS) {
    const int ns = std::min(kWS, tb - s0), nt = (ns + 7) / 8;
    cudaError_t e = cudaSuccess;
#define GPK_G2S(NTV)                                                                                           \
  case NTV:                                                                                                    \
    e = vec ? g2s_launch<true, NTV>(st, C, ldc, ka, W, ldw, s0, ns, n, Z, R, ldn, sig2, prz, pzz)               \
            : g2s_launch<false, NTV>(st, C, ldc, ka, W, ldw, s0, ns, n, Z, R, ldn, sig2, prz, pzz);             \
    break;
    switch (nt) {
      GPK_G2S(1) GPK_G2S(2) GPK_G2S(3) GPK_G2S(4) GPK_G2S(5) GPK_G2S(6) GPK_G2S(7) GPK_G2S(8)
    }
#undef GPK_G2S
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_cg_beta_p(double* P, const double* Z, int n, long long ldn, int t, SlotState* ss,
                             const double* prz, const double* pzz, unsigned* cnt, int k, double rel_tol,
                             double* beta_hist, double* resid_hist, int max_iters, unsigned long long* vmax,
                             SlotState* snap, cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  int bx = (n + 4 * kWT - 1) / (4 * kWT);
  if (bx > 32) bx = 32;
  cg_beta_p_kernel<<<dim3(bx, t), kWT, 0, st>>>(P, Z, n, ldn, ss, prz, pzz, wood_grid(), cnt, k, rel_tol, beta_hist,
                                                resid_hist, max_iters, vmax, snap);
  return cudaGetLastError();
}

// ===========================================================================
// The whole CG vector phase of one iteration as ONE cooperative launch (single rank,
// Woodbury preconditioner; krylov.hpp:76-119 + preconditioners.hpp:114-118):
//   1 pap partials over the CTA's rows      | grid barrier
//   2 alpha of column s in CTA s mod G      | grid barrier
//   3 x/r update fused into G1s (W = L^T r) | grid barrier
//   4 G1s partial reduction -> W            | grid barrier
//   5 G2s: z = (r - C W)/s2, r.z, z.z       | grid barrier
//   6 beta of column s in CTA s mod G, the slot state (+ pinned host snapshot)
//                                           | grid barrier
//   7 p = z + beta p on the CTA's rows, |p| column maxima for the next fp16 pack
// instead of five launches (pap+alpha, G1s, G1s reduce, G2s, beta+p) whose boundaries
// drained the GPU between phases (C2: 66 us per iteration, the work itself ~15 us of L2
// traffic).  Every phase keeps a fixed partition (rows_of over the G CTAs) and fixed-order
// reductions, so a column's arithmetic never depends on the other columns (batched ==
// independent, krylov.hpp:131-132) and reruns are bitwise reproducible.
// ===========================================================================
namespace cgrp = cooperative_groups;

GPK_DEV void alpha_step_c(SlotState& x, double pap, int k, double* alpha_hist, int max_iters) {
  if (x.flag != 0) {  // krylov.hpp:78-83 (cg_alpha_kernel's semantics)
    x.alpha = 0.0;
    return;
  }
  const double alpha = x.rz / pap;
  x.alpha = alpha;
  if (!isfinite(alpha) || alpha <= 0.0) {
    x.status = kStatusAlpha;
    x.bad = alpha;
    x.iters = k;
    x.flag = kFlagError;
    x.alpha = 0.0;
    return;
  }
  if (alpha_hist) alpha_hist[static_cast<long long>(x.col) * max_iters + (k - 1)] = alpha;
}

struct CoopArgs {
  const double* L;
  const double* Cm;
  long long ldl, ldc;
  int ka;
  double *X, *R, *P, *Z;
  const double* Y;
  long long ldn;
  int tb, n;
  double sig2, psig2;
  double *ppap, *pg1, *W, *prz, *pzz;
  SlotState* ss;
  int k;
  double rel_tol;
  double *ahist, *bhist, *rhist;
  int max_iters;
  unsigned long long* vmax;
  SlotState* snap;
};

template <bool VEC>
__global__ void __launch_bounds__(kWT, 2) cg_iter_coop_kernel(CoopArgs a) {
  extern __shared__ __align__(16) double wsm[];
  __shared__ double s_al[kWS];
  __shared__ double srz[8][kWS], szz[8][kWS];
  __shared__ double red8[8][32];
  __shared__ double red[kWT / 32];
  cgrp::grid_group grid = cgrp::this_grid();
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  int r0, r1;
  rows_of(b, G, a.n, r0, r1);
  // 1. p.(Kp + s2 p) over the CTA's rows: warp per column, lane-strided rows + butterfly
  for (int s = w; s < a.tb; s += kWT / 32) {
    const double* p = a.P + s * a.ldn;
    const double* y = a.Y + s * a.ldn;
    double acc = 0.0;
    for (int i = r0 + lane; i < r1; i += 32) {
      const double pv = p[i];
      acc += pv * (y[i] + a.sig2 * pv);
    }
    acc = warp_sum(acc);
    if (lane == 0) a.ppap[static_cast<long long>(s) * G + b] = acc;
  }
  grid.sync();
  // 2. alpha (krylov.hpp:78-83); the fp16 pack's column maxima are re-armed here
  for (int s = b; s < a.tb; s += G) {
    double acc = 0.0;
    for (int c = tid; c < G; c += kWT) acc += __ldcg(a.ppap + static_cast<long long>(s) * G + c);
    const double pap = block_sum(acc, red);
    if (tid == 0) {
      SlotState x = a.ss[s];
      alpha_step_c(x, pap, a.k, a.ahist, a.max_iters);
      a.ss[s] = x;
      if (a.vmax) a.vmax[s] = 0ull;
    }
  }
  grid.sync();
  // 3. x += alpha p, r -= alpha (Kp + s2 p) fused into G1s partials of W = L^T r
  for (int s0 = 0; s0 < a.tb; s0 += kWS) {
    const int nt = (min(kWS, a.tb - s0) + 7) / 8;
    __syncthreads();
#define GPK_G1C(NTV)                                                                                          \
  case NTV:                                                                                                   \
    g1s_group<true, VEC, NTV>(b, G, s0, a.L, a.ldl, a.ka, a.R, a.ldn, a.tb, a.n, a.pg1, a.X, a.P, a.Y, a.sig2, \
                              a.ss, wsm, s_al);                                                               \
    break;
    switch (nt) { GPK_G1C(1) GPK_G1C(2) GPK_G1C(3) GPK_G1C(4) GPK_G1C(5) GPK_G1C(6) GPK_G1C(7) GPK_G1C(8) }
#undef GPK_G1C
  }
  grid.sync();
  // 4. W = sum of the G partials in fixed order
  {
    const long long tot = static_cast<long long>(a.ka) * a.tb, nch = (tot + 31) / 32;
    for (long long c = b; c < nch; c += G) {
      __syncthreads();
      g1s_reduce_chunk(c, a.pg1, G, a.ka, a.tb, a.W, a.ka, red8);
    }
  }
  grid.sync();
  // 5. z = (r - C W) / s2 and the CTA's r.z / z.z partials
  for (int s0 = 0; s0 < a.tb; s0 += kWS) {
    const int ns = min(kWS, a.tb - s0), nt = (ns + 7) / 8;
    __syncthreads();
#define GPK_G2C(NTV)                                                                                            \
  case NTV:                                                                                                     \
    g2s_group<VEC, NTV>(b, G, a.Cm, a.ldc, a.ka, a.W, a.ka, s0, ns, a.n, a.Z, a.R, a.ldn, a.psig2, a.prz, a.pzz, \
                        wsm, srz, szz);                                                                         \
    break;
    switch (nt) { GPK_G2C(1) GPK_G2C(2) GPK_G2C(3) GPK_G2C(4) GPK_G2C(5) GPK_G2C(6) GPK_G2C(7) GPK_G2C(8) }
#undef GPK_G2C
  }
  grid.sync();
  // 6. beta (krylov.hpp:96-119) and the slot state (+ the host's pinned snapshot)
  for (int s = b; s < a.tb; s += G) {
    double ar = 0.0, az = 0.0;
    for (int c = tid; c < G; c += kWT) {
      ar += __ldcg(a.prz + static_cast<long long>(s) * G + c);
      az += __ldcg(a.pzz + static_cast<long long>(s) * G + c);
    }
    const double rz_new = block_sum(ar, red);
    const double zz = block_sum(az, red);
    if (tid == 0) {
      SlotState x = a.ss[s];
      beta_step_s(x, rz_new, zz, a.k, a.rel_tol, a.bhist, a.rhist, a.max_iters);
      a.ss[s] = x;
      if (a.snap) a.snap[s] = x;
    }
  }
  grid.sync();
  // 7. p = z + beta p on the CTA's rows (krylov.hpp:116) and |p| column maxima
  for (int s = w; s < a.tb; s += kWT / 32) {
    const SlotState* x = a.ss + s;
    const bool live = __ldcg(&x->flag) == 0;
    const double beta = __ldcg(&x->beta);
    double* p = a.P + s * a.ldn;
    const double* z = a.Z + s * a.ldn;
    double mx = 0.0;
    for (int i = r0 + lane; i < r1; i += 32) {
      double pv = p[i];
      if (live) {
        pv = z[i] + beta * pv;
        p[i] = pv;
      }
      mx = fmax(mx, fabs(pv));
    }
    if (a.vmax) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0 && mx > 0.0) atomicMax(a.vmax + s, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
  }
}

namespace {
template <bool VEC>
int coop_grid() {
  static int g = [] {
    cudaFuncSetAttribute(cg_iter_coop_kernel<VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kWSmem));
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cg_iter_coop_kernel<VEC>, kWT, kWSmem);
    return std::min(per, 2) * sm_count();
  }();
  return g;
}
}  // namespace

bool cg_iter_coop_available() {
  static bool ok = [] {
    // opt-in (GPK_COOP=1): measured SLOWER than the five-launch path at C2 (0.102 vs 0.079 ms per
    // iteration, profiles/r2_coop_vector_phase.txt): the warp-per-column phases and the five grid
    // barriers of 296 CTAs cost more than the kernel boundaries they replace
    const char* e = std::getenv("GPK_COOP");
    if (!(e && e[0] == '1')) return false;
    return coop_grid<true>() >= sm_count() && coop_grid<false>() >= sm_count();
  }();
  return ok;
}

cudaError_t launch_cg_iter_coop(const double* L, long long ldl, const double* Cm, long long ldc, int ka, double* X,
                                double* R, double* P, double* Z, const double* Y, long long ldn, int tb, int n,
                                double sig2, double psig2, double* ppap, double* pg1, double* W, double* prz,
                                double* pzz, SlotState* ss, int k, double rel_tol, double* ahist, double* bhist,
                                double* rhist, int max_iters, unsigned long long* vmax, SlotState* snap,
                                cudaStream_t st) {
  if (tb <= 0) return cudaSuccess;
  CoopArgs a{L, Cm, ldl, ldc, ka, X, R, P, Z, Y, ldn, tb, n, sig2, psig2, ppap, pg1, W, prz, pzz, ss, k,
             rel_tol, ahist, bhist, rhist, max_iters, vmax, snap};
  const bool vec = aligned16(L) && aligned16(R) && aligned16(Cm) && aligned16(W) && ldl % 2 == 0 && ldn % 2 == 0 &&
                   ldc % 2 == 0 && ka % 2 == 0;
  void* args[] = {&a};
  const int G = vec ? coop_grid<true>() : coop_grid<false>();
  const void* fn = vec ? reinterpret_cast<const void*>(cg_iter_coop_kernel<true>)
                       : reinterpret_cast<const void*>(cg_iter_coop_kernel<false>);
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kWT), args, kWSmem, st);
}

}  // namespace gpk
