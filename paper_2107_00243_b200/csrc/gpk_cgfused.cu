// Fused mBCG iteration kernels (single-rank path).  One CG iteration of
// krylov.hpp:76-119 for all active columns runs as
//   pack V -> fused kernel MVM -> [pap dots + alpha] -> [x/r update + L^T r] ->
//   L^T r chunk reduction -> [Woodbury z + r.z / z.z + beta] -> [p update + |p| column max]
// instead of twelve launches: grid-wide reductions finish in the LAST CTA to arrive
// (threadfence + per-column arrival counter, the counter re-armed by that CTA), so the
// scalar steps need no launches of their own.  Every reduction keeps a fixed partition
// and a fixed order (deterministic; a column never depends on the others).
#include <cfloat>

#include "gpk_common.cuh"
#include "gpk_linalg.h"

namespace gpk {

constexpr int kVT = 256;
constexpr int kRB = 1024;

GPK_DEV double reduce_chunks_cg(const double* part, int nrb, double* red) {
  double acc = 0.0;
  for (int c = threadIdx.x; c < nrb; c += blockDim.x) acc += __ldcg(part + c);
  return block_sum(acc, red);
}

// alpha step of krylov.hpp:78-83 (shared with cg_alpha_kernel's semantics)
GPK_DEV void alpha_step(SlotState& x, double pap, int k, double* alpha_hist, int max_iters) {
  if (x.flag != 0) {
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

// beta step of krylov.hpp:94-119
GPK_DEV void beta_step(SlotState& x, double rz_new, double zz, int k, double rel_tol, double* beta_hist,
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

// ---- F1: per-chunk p.(Kp + s2 p) partials (dot_partials_kernel<1> partition) + alpha in
// the last chunk CTA of each column.  With `parts` the fused MVM's split-K partials are summed
// here (split order 0..S-1 from 0.0, exactly reduce_splits' sums) and Kp is stored for the
// x / r update: one launch and one pass over Kp less per iteration.
__global__ void cg_pap_alpha_kernel(const double* __restrict__ P, double* __restrict__ Y, double sig2, int n,
                                    long long ldn, int nrb, double* __restrict__ part, unsigned* __restrict__ cnt,
                                    int k, SlotState* __restrict__ ss, double* __restrict__ alpha_hist,
                                    int max_iters, unsigned long long* __restrict__ vmax,
                                    const double* __restrict__ parts, int splits, long long sstride, long long ldp) {
  __shared__ double red[kVT / 32];
  __shared__ bool last;
  const int s = blockIdx.y, b = blockIdx.x;
  const double* a = P + s * ldn;
  double* y = Y + s * ldn;
  double acc = 0.0;
  if (parts != nullptr) {
    const double* ps = parts + s * ldp + b * kRB + threadIdx.x;
    constexpr int Q = kRB / kVT;
    double yi[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) yi[q] = 0.0;
#pragma unroll 4
    for (int sp = 0; sp < splits; ++sp) {  // Q x 4 independent L2 loads in flight
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (b * kRB + q * kVT + threadIdx.x < n) yi[q] += __ldcg(ps + sp * sstride + q * kVT);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = b * kRB + q * kVT + threadIdx.x;
      if (i < n) {
        y[i] = yi[q];
        acc += a[i] * (yi[q] + sig2 * a[i]);
      }
    }
  } else {
    for (int q = 0; q < kRB / kVT; ++q) {
      const int i = b * kRB + q * kVT + threadIdx.x;
      if (i < n) acc += a[i] * (y[i] + sig2 * a[i]);
    }
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) {
    part[static_cast<long long>(s) * nrb + b] = t;
    __threadfence();
    last = atomicAdd(cnt + s, 1u) == static_cast<unsigned>(nrb - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double pap = reduce_chunks_cg(part + static_cast<long long>(s) * nrb, nrb, red);
  if (threadIdx.x == 0) {
    alpha_step(ss[s], pap, k, alpha_hist, max_iters);
    if (vmax) vmax[s] = 0ull;
    cnt[s] = 0;
  }
}

cudaError_t launch_cg_pap_alpha(const double* P, double* Y, double sig2, int n, long long ldn, int t,
                                double* part, unsigned* cnt, int k, SlotState* ss, double* alpha_hist, int max_iters,
                                cudaStream_t st, unsigned long long* vmax, const double* parts, int splits,
                                long long sstride, long long ldp) {
  if (t <= 0) return cudaSuccess;
  const int nrb = (n + kRB - 1) / kRB;
  cg_pap_alpha_kernel<<<dim3(nrb, t), kVT, 0, st>>>(P, Y, sig2, n, ldn, nrb, part, cnt, k, ss, alpha_hist,
                                                    max_iters, vmax, splits > 1 ? parts : nullptr, splits, sstride,
                                                    ldp);
  return cudaGetLastError();
}

// ---- F2: x += alpha p, r -= alpha (Kp + s2 p) fused into the G1 product W = L^T r_new
// (g1_kernel's DMMA structure and chunk partition; r_new is formed in registers by every
// CTA that needs it and stored, with x, by warp 0 of the k-group-0 CTAs only -- into a
// second buffer Rn, since other CTAs still read the old r).
GPK_DEV void dmma884f(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) g1_xr_kernel(const double* __restrict__ A, long long lda, int ka,
                                                    double* __restrict__ X, const double* __restrict__ R,
                                                    double* __restrict__ Rn, const double* __restrict__ P,
                                                    const double* __restrict__ Y,
                                                    double sig2, long long ldn, int tb, int n, int ch,
                                                    const SlotState* __restrict__ ss, double* __restrict__ part) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.y * 8 + w;
  const bool writer = blockIdx.y == 0 && w == 0;
  if (mt * 8 >= ka && !writer) return;  // warp-uniform; no block-level synchronisation below
  const int chunk = blockIdx.x;
  const int n0 = blockIdx.z * 64;
  const int r = lane & 3, m = lane >> 2;
  const int kk = mt * 8 + m;
  const bool aval = kk < ka;
  const double* acol = A + static_cast<long long>(aval ? kk : 0) * lda;
  long long boff[8];
  bool bval[8], live[8];
  double al[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int sj = n0 + 8 * j + m;
    bval[j] = sj < tb;
    boff[j] = static_cast<long long>(bval[j] ? sj : 0) * ldn;
    const SlotState& x = ss[bval[j] ? sj : 0];
    live[j] = bval[j] && x.flag == 0;
    al[j] = live[j] ? x.alpha : 0.0;
  }
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int i0 = chunk * ch;
  const int i1 = min(n, i0 + ch);
  for (int ib = i0; ib < i1; ib += 16) {
    double av[4], bv[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int row = ib + 4 * u + r;
      const bool rv = row < i1;
      av[u] = (aval && rv) ? acol[row] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double v = 0.0;
        if (bval[j] && rv) {
          const long long o = boff[j] + row;
          v = R[o];
          if (live[j]) {  // krylov.hpp:94-95 (cg_update_xr_kernel's expressions)
            const double p = P[o];
            const double ap = Y[o] + sig2 * p;
            v -= al[j] * ap;
            if (writer) X[o] += al[j] * p;
          }
          if (writer) Rn[o] = v;
        }
        bv[u][j] = v;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma884f(acc[j], av[u], bv[u][j]);
  }
  if (mt * 8 >= ka) return;
  const int kko = mt * 8 + m;
  if (kko < ka) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int s = n0 + 8 * j + 2 * r + e;
        if (s < tb) part[(static_cast<long long>(chunk) * tb + s) * ka + kko] = acc[j][e];
      }
  }
}

// ---- F3: Woodbury z = (r - C W) / s2 (g2_kernel structure) + per-64-row r.z, z.z partials
// + beta in the last CTA of each 64-column group; that CTA also clears the |p| maxima of
// its columns for F4.
__global__ void __launch_bounds__(256) g2_dots_beta_kernel(
    const double* __restrict__ A, long long lda, int ka, const double* __restrict__ W, long long ldw, int tb, int n,
    double* __restrict__ Z, const double* __restrict__ R, long long ldn, double sig2, double* __restrict__ prz,
    double* __restrict__ pzz, unsigned* __restrict__ cnt, int k, double rel_tol, SlotState* __restrict__ ss,
    double* __restrict__ beta_hist, double* __restrict__ resid_hist, int max_iters,
    unsigned long long* __restrict__ vmax) {
  __shared__ double srz[8][64], szz[8][64];
  __shared__ bool last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = (blockIdx.x * 8 + w) * 8;
  const int n0 = blockIdx.y * 64;
  const int r = lane & 3, m = lane >> 2;
  const int row = i0 + m;
  const bool rowv = row < n;
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  if (i0 < n) {
    const double* arow = A + (rowv ? row : 0);
    const double* wcol[8];
    bool wval[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int sj = n0 + 8 * j + m;
      wval[j] = sj < tb;
      wcol[j] = W + static_cast<long long>(wval[j] ? sj : 0) * ldw;
    }
    for (int kb = 0; kb < ka; kb += 16) {
      double av[4], bv[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kr = kb + 4 * u + r;
        const bool kv = kr < ka;
        av[u] = (kv && rowv) ? arow[static_cast<long long>(kr) * lda] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) bv[u][j] = (kv && wval[j]) ? wcol[j][kr] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma884f(acc[j], av[u], bv[u][j]);
    }
  }
  // z, then the lane's r.z / z.z contributions (row `row`, columns n0 + 8j + 2r + e)
  double crz[8][2], czz[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int s = n0 + 8 * j + 2 * r + e;
      crz[j][e] = czz[j][e] = 0.0;
      if (rowv && s < tb) {
        const long long o = static_cast<long long>(s) * ldn + row;
        const double rr = R[o];
        const double z = rr / sig2 - acc[j][e] / sig2;  // preconditioners.hpp:114-118
        Z[o] = z;
        crz[j][e] = rr * z;
        czz[j][e] = z * z;
      }
    }
  // sum over the warp's 8 rows (lanes with equal r), fixed butterfly
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        crz[j][e] += __shfl_xor_sync(0xffffffffu, crz[j][e], o);
        czz[j][e] += __shfl_xor_sync(0xffffffffu, czz[j][e], o);
      }
  if (m == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        srz[w][8 * j + 2 * r + e] = crz[j][e];
        szz[w][8 * j + 2 * r + e] = czz[j][e];
      }
  }
  __syncthreads();
  const int nbx = gridDim.x;
  if (threadIdx.x < 64) {
    const int c = threadIdx.x, s = n0 + c;
    double a = 0.0, b = 0.0;
    for (int q = 0; q < 8; ++q) {  // the CTA's 64 rows in warp order
      a += srz[q][c];
      b += szz[q][c];
    }
    if (s < tb) {
      prz[static_cast<long long>(s) * nbx + blockIdx.x] = a;
      pzz[static_cast<long long>(s) * nbx + blockIdx.x] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(cnt + blockIdx.y, 1u) == static_cast<unsigned>(nbx - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int ncol = min(64, tb - n0);
  for (int c = w; c < ncol; c += 8) {  // one warp per column: fixed lane-strided sums + butterfly
    const int s = n0 + c;
    double rz = 0.0, zz = 0.0;
    for (int b = lane; b < nbx; b += 32) {
      rz += __ldcg(prz + static_cast<long long>(s) * nbx + b);
      zz += __ldcg(pzz + static_cast<long long>(s) * nbx + b);
    }
    rz = warp_sum(rz);
    zz = warp_sum(zz);
    if (lane == 0) {
      beta_step(ss[s], rz, zz, k, rel_tol, beta_hist, resid_hist, max_iters);
      if (vmax) vmax[s] = 0ull;
    }
  }
  if (threadIdx.x == 0) cnt[blockIdx.y] = 0;
}

int g2_row_blocks(int n) { return (n + 63) / 64; }

cudaError_t launch_g1_xr(const double* L, long long ldl, int ka, double* X, const double* R, double* Rn,
                         const double* P, const double* Y, double sig2, long long ldn, int tb, int n,
                         const SlotState* ss, double* part, double* W, long long ldw, cudaStream_t st) {
  if (ka <= 0 || tb <= 0) return cudaSuccess;
  const int ch = g1_chunk_rows(n, ka);
  const int nch = (n + ch - 1) / ch;
  dim3 g(nch, (ka + 63) / 64, (tb + 63) / 64);
  g1_xr_kernel<<<g, 256, 0, st>>>(L, ldl, ka, X, R, Rn, P, Y, sig2, ldn, tb, n, ch, ss, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_g1_reduce(part, n, ka, tb, W, ldw, st);
}

cudaError_t launch_g2_dots_beta(const double* C, long long ldc, int ka, const double* W, long long ldw, int tb, int n,
                                double* Z, const double* R, long long ldn, double sig2, double* prz, double* pzz,
                                unsigned* cnt, int k, double rel_tol, SlotState* ss, double* beta_hist,
                                double* resid_hist, int max_iters, unsigned long long* vmax, cudaStream_t st) {
  if (tb <= 0) return cudaSuccess;
  dim3 g(g2_row_blocks(n), (tb + 63) / 64);
  g2_dots_beta_kernel<<<g, 256, 0, st>>>(C, ldc, ka, W, ldw, tb, n, Z, R, ldn, sig2, prz, pzz, cnt, k, rel_tol, ss,
                                         beta_hist, resid_hist, max_iters, vmax);
  return cudaGetLastError();
}

// ---- F4: p = z + beta p (live columns) and max |p| per column for the next fp16 pack
__global__ void cg_p_vmax_kernel(double* __restrict__ P, const double* __restrict__ Z, int n, long long ldn,
                                 const SlotState* __restrict__ ss, unsigned long long* __restrict__ vmax) {
  const int s = blockIdx.y;
  const SlotState& x = ss[s];
  const bool live = x.flag == 0;
  const double beta = x.beta;
  double mx = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const long long o = s * ldn + i;
    double p = P[o];
    if (live) {
      p = Z[o] + beta * p;  // krylov.hpp:116 (cg_update_p_kernel's expression)
      P[o] = p;
    }
    mx = fmax(mx, fabs(p));
  }
  if (vmax) {  // CTA maximum first: one atomic per CTA (order-independent, so deterministic)
    __shared__ double wm[kVT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < kVT / 32; ++q) mx = fmax(mx, wm[q]);
      if (mx > 0.0) atomicMax(vmax + s, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
  }
}

cudaError_t launch_cg_p_vmax(double* P, const double* Z, int n, long long ldn, int t, const SlotState* ss,
                             unsigned long long* vmax, cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  int bx = (n + 4 * kVT - 1) / (4 * kVT);
  if (bx > 32) bx = 32;
  cg_p_vmax_kernel<<<dim3(bx, t), kVT, 0, st>>>(P, Z, n, ldn, ss, vmax);
  return cudaGetLastError();
}

}  // namespace gpk
