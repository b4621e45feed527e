// mBCG vector kernels, Woodbury skinny GEMMs, pivoted Cholesky (fp64).
//
// All n-length state is fp64, column-major [slot][ldn].  Every reduction uses a
// fixed partition of rows into 1024-row chunks and a fixed tree, so results are
// deterministic and a column's value never depends on the other columns of the
// block (batched_pcg contract, krylov.hpp:131-132).
#include <algorithm>
#include <cfloat>

#include "gpk_common.cuh"
#include "gpk_linalg.h"

namespace gpk {

constexpr int kRB = 1024;  // rows per reduction chunk
constexpr int kVT = 256;   // threads per vector-kernel block

// ---------------------------------------------------------------------------
// per-column dot partials:  part[slot][chunk] = sum_{i in chunk} f(i, slot)
// ---------------------------------------------------------------------------
template <int OP>
__global__ void dot_partials_kernel(const double* __restrict__ A, const double* __restrict__ B, double sig2, int n,
                                    long long ldn, int nrb, double* __restrict__ part) {
  __shared__ double red[kVT / 32];
  const int s = blockIdx.y;
  const int b = blockIdx.x;
  const double* a = A + s * ldn;
  const double* bb = B + s * ldn;
  double acc = 0.0;
  for (int q = 0; q < kRB / kVT; ++q) {
    const int i = b * kRB + q * kVT + threadIdx.x;
    if (i < n) {
      if constexpr (OP == 0) acc += a[i] * bb[i];                        // a . b
      if constexpr (OP == 1) acc += a[i] * (bb[i] + sig2 * a[i]);        // p . (K p + s2 p)
    }
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) part[static_cast<long long>(s) * nrb + b] = t;
}

// total[slot] = sum over chunks in a fixed tree
GPK_DEV double reduce_chunks(const double* __restrict__ part, int nrb, double* red) {
  double acc = 0.0;
  for (int c = threadIdx.x; c < nrb; c += blockDim.x) acc += part[c];
  return block_sum(acc, red);
}

int num_chunks(int n) { return (n + kRB - 1) / kRB; }

cudaError_t launch_dot_partials(int op, const double* A, const double* B, double sig2, int n, long long ldn, int t,
                                double* part, cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  dim3 g(num_chunks(n), t);
  if (op == 0) dot_partials_kernel<0><<<g, kVT, 0, st>>>(A, B, sig2, n, ldn, g.x, part);
  else dot_partials_kernel<1><<<g, kVT, 0, st>>>(A, B, sig2, n, ldn, g.x, part);
  return cudaGetLastError();
}

__global__ void reduce_partials_kernel(const double* __restrict__ part, int nrb, double* __restrict__ out) {
  __shared__ double red[kVT / 32];
  const double v = reduce_chunks(part + static_cast<long long>(blockIdx.x) * nrb, nrb, red);
  if (threadIdx.x == 0) out[blockIdx.x] = v;
}

cudaError_t launch_reduce_partials(const double* part, int nrb, int t, double* out, cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  reduce_partials_kernel<<<t, kVT, 0, st>>>(part, nrb, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// CG scalar steps (krylov.hpp:76-119), one block per active slot
// ---------------------------------------------------------------------------
__global__ void cg_init_kernel(const double* __restrict__ part_rz, const double* __restrict__ part_zz, int nrb,
                               SlotState* __restrict__ ss) {
  __shared__ double red[kVT / 32];
  const int s = blockIdx.x;
  const double rz = reduce_chunks(part_rz + static_cast<long long>(s) * nrb, nrb, red);
  const double zz = reduce_chunks(part_zz + static_cast<long long>(s) * nrb, nrb, red);
  if (threadIdx.x == 0) {
    SlotState& x = ss[s];
    x.rz = rz;
    x.norm0 = sqrt(zz);  // ||P^{-1} b|| (krylov.hpp:59-60)
    x.pres = x.norm0;
    x.iters = 0;
    x.status = 0;
    x.alpha_prev = 0.0;
    x.beta_prev = 0.0;
    x.flag = (x.norm0 == 0.0) ? kFlagConverged : 0;  // zero rhs: converged, 0 iterations (:61-64)
    x.alpha = 0.0;
  }
}

__global__ void cg_alpha_kernel(const double* __restrict__ part_pap, int nrb, int k, SlotState* __restrict__ ss,
                                double* __restrict__ alpha_hist, int max_iters) {
  __shared__ double red[kVT / 32];
  const int s = blockIdx.x;
  const double pap = reduce_chunks(part_pap + static_cast<long long>(s) * nrb, nrb, red);
  if (threadIdx.x == 0) {
    SlotState& x = ss[s];
    if (x.flag != 0) {  // converged / failed columns stay frozen until the host compacts them out
      x.alpha = 0.0;
      return;
    }
    const double alpha = x.rz / pap;
    x.alpha = alpha;
    if (!isfinite(alpha) || alpha <= 0.0) {  // krylov.hpp:79-83
      x.status = kStatusAlpha;
      x.bad = alpha;
      x.iters = k;
      x.flag = kFlagError;
      x.alpha = 0.0;  // freeze the column
      return;
    }
    if (alpha_hist) alpha_hist[static_cast<long long>(x.col) * max_iters + (k - 1)] = alpha;
  }
}

__global__ void cg_beta_kernel(const double* __restrict__ part_rz, const double* __restrict__ part_zz, int nrb,
                               int k, double rel_tol, SlotState* __restrict__ ss, double* __restrict__ beta_hist,
                               double* __restrict__ resid_hist, int max_iters) {
  __shared__ double red[kVT / 32];
  const int s = blockIdx.x;
  const double rz_new = reduce_chunks(part_rz + static_cast<long long>(s) * nrb, nrb, red);
  const double zz = reduce_chunks(part_zz + static_cast<long long>(s) * nrb, nrb, red);
  if (threadIdx.x == 0) {
    SlotState& x = ss[s];
    if (x.flag != 0) {
      x.beta = 0.0;
      return;
    }
    if (!isfinite(rz_new) || rz_new < 0.0) {  // krylov.hpp:97-100
      x.status = kStatusRz;
      x.bad = rz_new;
      x.iters = k;
      x.flag = kFlagError;
      x.beta = 0.0;
      return;
    }
    const double pres = sqrt(zz);  // :102
    const long long base = static_cast<long long>(x.col) * max_iters + (k - 1);
    if (resid_hist) resid_hist[base] = pres;
    x.iters = k;
    x.pres = pres;
    if (pres <= rel_tol * x.norm0 || rz_new == 0.0) {  // :106-113
      x.flag = kFlagConverged;
      x.beta = 0.0;
      return;
    }
    const double beta = rz_new / x.rz;  // :115
    if (beta_hist) beta_hist[base] = beta;
    x.beta = beta;
    x.rz = rz_new;
  }
}

// x += alpha p ; r -= alpha (Kp + s2 p)     (krylov.hpp:94-95)
__global__ void cg_update_xr_kernel(double* __restrict__ X, double* __restrict__ R, const double* __restrict__ P,
                                    const double* __restrict__ Y, double sig2, int n, long long ldn,
                                    const SlotState* __restrict__ ss) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const SlotState& x = ss[s];
  if (x.flag != 0) return;
  const double a = x.alpha;
  const long long o = s * ldn + i;
  const double p = P[o];
  const double ap = Y[o] + sig2 * p;
  X[o] += a * p;
  R[o] -= a * ap;
}

// p = z + beta p  for slots that keep iterating   (krylov.hpp:116)
__global__ void cg_update_p_kernel(double* __restrict__ P, const double* __restrict__ Z, int n, long long ldn,
                                   const SlotState* __restrict__ ss) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const SlotState& x = ss[s];
  if (x.flag != 0) return;
  const long long o = s * ldn + i;
  P[o] = Z[o] + x.beta * P[o];
}

cudaError_t launch_cg_init(const double* part_rz, const double* part_zz, int nrb, int t, SlotState* ss,
                           cudaStream_t st) {
  cg_init_kernel<<<t, kVT, 0, st>>>(part_rz, part_zz, nrb, ss);
  return cudaGetLastError();
}
cudaError_t launch_cg_alpha(const double* part, int nrb, int t, int k, SlotState* ss, double* alpha_hist,
                            int max_iters, cudaStream_t st) {
  cg_alpha_kernel<<<t, kVT, 0, st>>>(part, nrb, k, ss, alpha_hist, max_iters);
  return cudaGetLastError();
}
cudaError_t launch_cg_beta(const double* part_rz, const double* part_zz, int nrb, int t, int k, double rel_tol,
                           SlotState* ss, double* beta_hist, double* resid_hist, int max_iters, cudaStream_t st) {
  cg_beta_kernel<<<t, kVT, 0, st>>>(part_rz, part_zz, nrb, k, rel_tol, ss, beta_hist, resid_hist, max_iters);
  return cudaGetLastError();
}
cudaError_t launch_cg_update_xr(double* X, double* R, const double* P, const double* Y, double sig2, int n,
                                long long ldn, int t, const SlotState* ss, cudaStream_t st) {
  dim3 g((n + kVT - 1) / kVT, t);
  cg_update_xr_kernel<<<g, kVT, 0, st>>>(X, R, P, Y, sig2, n, ldn, ss);
  return cudaGetLastError();
}
cudaError_t launch_cg_update_p(double* P, const double* Z, int n, long long ldn, int t, const SlotState* ss,
                               cudaStream_t st) {
  dim3 g((n + kVT - 1) / kVT, t);
  cg_update_p_kernel<<<g, kVT, 0, st>>>(P, Z, n, ldn, ss);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// elementwise helpers
// ---------------------------------------------------------------------------
// dst[s][i] = src[map ? map[s] : s][i] * scale (gather + scale), or zero when src is null
__global__ void gather_cols_kernel(const double* __restrict__ src, long long lds, const int* __restrict__ map,
                                   double scale, int n, double* __restrict__ dst, long long ldd) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 0.0;
  if (src) v = src[static_cast<long long>(map ? map[s] : s) * lds + i] * scale;
  dst[static_cast<long long>(s) * ldd + i] = v;
}
cudaError_t launch_gather_cols(const double* src, long long lds, const int* map, double scale, int n, int t,
                               double* dst, long long ldd, cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  dim3 g((n + kVT - 1) / kVT, t);
  gather_cols_kernel<<<g, kVT, 0, st>>>(src, lds, map, scale, n, dst, ldd);
  return cudaGetLastError();
}
// dst[map[s]][i] = src[s][i] (scatter)
__global__ void scatter_cols_kernel(const double* __restrict__ src, long long lds, const int* __restrict__ map, int n,
                                    double* __restrict__ dst, long long ldd) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dst[static_cast<long long>(map[s]) * ldd + i] = src[static_cast<long long>(s) * lds + i];
}
cudaError_t launch_scatter_cols(const double* src, long long lds, const int* map, int n, int t, double* dst,
                                long long ldd, cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  dim3 g((n + kVT - 1) / kVT, t);
  scatter_cols_kernel<<<g, kVT, 0, st>>>(src, lds, map, n, dst, ldd);
  return cudaGetLastError();
}
// a = alpha*a + beta*b (elementwise over t columns)
__global__ void axpby_kernel(double* __restrict__ a, const double* __restrict__ b, double alpha, double beta, int n,
                             long long ld) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long o = s * ld + i;
  a[o] = alpha * a[o] + beta * b[o];
}
cudaError_t launch_axpby(double* a, const double* b, double alpha, double beta, int n, int t, long long ld,
                         cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  dim3 g((n + kVT - 1) / kVT, t);
  axpby_kernel<<<g, kVT, 0, st>>>(a, b, alpha, beta, n, ld);
  return cudaGetLastError();
}
// Woodbury finish (preconditioners.hpp:114-118): z = r / s2 - T / s2  (T = C (L^T r))
__global__ void woodbury_finish_kernel(const double* __restrict__ R, const double* __restrict__ T, double sig2, int n,
                                       long long ldn, double* __restrict__ Z) {
  const int s = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long o = s * ldn + i;
  const double r = R[o] / sig2;
  Z[o] = T ? r - T[o] / sig2 : r;
}
cudaError_t launch_woodbury_finish(const double* R, const double* T, double sig2, int n, long long ldn, int t,
                                   double* Z, cudaStream_t st) {
  if (t <= 0) return cudaSuccess;
  dim3 g((n + kVT - 1) / kVT, t);
  woodbury_finish_kernel<<<g, kVT, 0, st>>>(R, T, sig2, n, ldn, Z);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Skinny fp64 GEMMs for the Woodbury solve, Gram matrix and trace terms, on the
// fp64 tensor cores (DMMA 8x8x4, mma.sync .f64):
//   G1: W[s][kk] = sum_i A[kk][i] * B[s][i]     (A^T B, A: [ka][lda], B: [tb][ldb])
//       per row-chunk partials (chunk = f(n) only), then a fixed-order chunk reduction.
//   G2: T[s][i]  = sum_kk A[kk][i] * W[s][kk]   (A W), optionally fused with the
//       Woodbury finish Z = R / s2 - T / s2.
// Each warp owns one 8-row m-tile and eight 8-column n-tiles (64 columns) and walks
// K in steps of 4 in a fixed order, so every output column is computed from its own
// column of B / W only (the batched == independent contract) and runs are bitwise
// reproducible.  Fragments come straight from global memory (L2-resident operands;
// every 32-byte sector fully used).
// ---------------------------------------------------------------------------
GPK_DEV void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// rows per G1 chunk: a function of n (~128 chunks), multiple of 16; for wide products
// (ka >= 512: the d+1 derivative factors of the backward pass, ka = (d+1) k) at most 32
// chunks, so the chunk partials (nch x ka x tb) stay well below the A operand's size
static int g1_chunk(int n, int ka = 0) {
  int ch = (n + 127) / 128;
  if (ka >= 512) ch = (n + 31) / 32;
  ch = (ch + 15) / 16 * 16;
  return ch < 64 ? 64 : ch;
}

__global__ void __launch_bounds__(256) g1_kernel(const double* __restrict__ A, long long lda, int ka,
                                                 const double* __restrict__ B, long long ldb, int tb, int n, int ch,
                                                 double* __restrict__ part) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.y * 8 + w;
  if (mt * 8 >= ka) return;  // warp-uniform; no block-level synchronisation below
  const int chunk = blockIdx.x;
  const int n0 = blockIdx.z * 64;
  const int r = lane & 3, m = lane >> 2;
  const int kk = mt * 8 + m;
  const bool aval = kk < ka;
  const double* acol = A + static_cast<long long>(aval ? kk : 0) * lda;
  const double* bcol[8];
  bool bval[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int sj = n0 + 8 * j + m;
    bval[j] = sj < tb;
    bcol[j] = B + static_cast<long long>(bval[j] ? sj : 0) * ldb;
  }
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int i0 = chunk * ch;
  const int i1 = min(n, i0 + ch);
  for (int ib = i0; ib < i1; ib += 16) {  // 4 k-steps per round: loads first, then the DMMAs
    double av[4], bv[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int row = ib + 4 * u + r;
      const bool rv = row < i1;
      av[u] = (aval && rv) ? acol[row] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) bv[u][j] = (bval[j] && rv) ? bcol[j][row] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma884(acc[j], av[u], bv[u][j]);
  }
  const int kko = mt * 8 + m;  // C fragment: row m, columns 2 r + e
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

// W[s][kk] = sum over chunks in fixed order: 4 threads per output (strided chunk
// subsets, 8-deep batched loads), combined in fixed order through shared memory.
__global__ void g1_reduce_kernel(const double* __restrict__ part, int nch, int ka, int tb, double* __restrict__ W,
                                 long long ldw) {
  __shared__ double red[4][64];
  const int q = threadIdx.x >> 6, o = threadIdx.x & 63;
  const long long idx = blockIdx.x * 64LL + o;
  const long long tot = static_cast<long long>(ka) * tb;
  double acc = 0.0;
  if (idx < tot) {
    const double* p = part + idx;
    const long long stride = tot;
    int c = q;
    for (; c + 28 < nch; c += 32) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = p[(c + 4 * u) * stride];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; c < nch; c += 4) acc += p[c * stride];
  }
  red[q][o] = acc;
  __syncthreads();
  if (q == 0 && idx < tot) {
    const int s = static_cast<int>(idx / ka), kk = static_cast<int>(idx % ka);
    W[s * ldw + kk] = ((red[0][o] + red[1][o]) + red[2][o]) + red[3][o];
  }
}

int g1_chunk_rows(int n, int ka) { return g1_chunk(n, ka); }

cudaError_t launch_g1_reduce(const double* part, int n, int ka, int tb, double* W, long long ldw, cudaStream_t st) {
  const int ch = g1_chunk(n, ka);
  const int nch = (n + ch - 1) / ch;
  const long long tot = static_cast<long long>(ka) * tb;
  g1_reduce_kernel<<<static_cast<unsigned>((tot + 63) / 64), 256, 0, st>>>(part, nch, ka, tb, W, ldw);
  return cudaGetLastError();
}

size_t g1_workspace(int n, int ka, int tb) {
  const int ch = g1_chunk(n, ka);
  return static_cast<size_t>((n + ch - 1) / ch) * ka * tb;
}

cudaError_t launch_g1(const double* A, long long lda, int ka, const double* B, long long ldb, int tb, int n,
                      double* part, double* W, long long ldw, cudaStream_t st) {
  if (ka <= 0 || tb <= 0) return cudaSuccess;
  const int ch = g1_chunk(n, ka);
  const int nch = (n + ch - 1) / ch;
  dim3 g(nch, (ka + 63) / 64, (tb + 63) / 64);
  g1_kernel<<<g, 256, 0, st>>>(A, lda, ka, B, ldb, tb, n, ch, part);
  const long long tot = static_cast<long long>(ka) * tb;
  g1_reduce_kernel<<<static_cast<unsigned>((tot + 63) / 64), 256, 0, st>>>(part, nch, ka, tb, W, ldw);
  return cudaGetLastError();
}

// G2 (+ Woodbury finish): warp = 8 rows x 64 columns, K = ka in steps of 4 (fixed order).
__global__ void __launch_bounds__(256) g2_kernel(const double* __restrict__ A, long long lda, int ka,
                                                 const double* __restrict__ W, long long ldw, int tb, int n,
                                                 double* __restrict__ T, long long ldt, const double* __restrict__ R,
                                                 long long ldr, double sig2) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = (blockIdx.x * 8 + w) * 8;
  if (i0 >= n) return;  // warp-uniform
  const int n0 = blockIdx.y * 64;
  const int r = lane & 3, m = lane >> 2;
  const int row = i0 + m;
  const bool rowv = row < n;
  const double* arow = A + (rowv ? row : 0);
  const double* wcol[8];
  bool wval[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int sj = n0 + 8 * j + m;
    wval[j] = sj < tb;
    wcol[j] = W + static_cast<long long>(wval[j] ? sj : 0) * ldw;
  }
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
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
      for (int j = 0; j < 8; ++j) dmma884(acc[j], av[u], bv[u][j]);
  }
  if (!rowv) return;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int s = n0 + 8 * j + 2 * r + e;
      if (s >= tb) continue;
      const long long o = static_cast<long long>(s) * ldt + row;
      if (R) T[o] = R[static_cast<long long>(s) * ldr + row] / sig2 - acc[j][e] / sig2;  // preconditioners.hpp:114-118
      else T[o] = acc[j][e];
    }
}

cudaError_t launch_g2(const double* A, long long lda, int ka, const double* W, long long ldw, int tb, int n,
                      double* T, long long ldt, cudaStream_t st) {
  if (tb <= 0) return cudaSuccess;
  dim3 g((n + 63) / 64, (tb + 63) / 64);
  g2_kernel<<<g, 256, 0, st>>>(A, lda, ka, W, ldw, tb, n, T, ldt, nullptr, 0, 1.0);
  return cudaGetLastError();
}

cudaError_t launch_woodbury_apply(const double* C, long long ldc, int ka, const double* W, long long ldw,
                                  const double* R, long long ldr, double sig2, int tb, int n, double* Z,
                                  long long ldz, cudaStream_t st) {
  if (tb <= 0) return cudaSuccess;
  dim3 g((n + 63) / 64, (tb + 63) / 64);
  g2_kernel<<<g, 256, 0, st>>>(C, ldc, ka, W, ldw, tb, n, Z, ldz, R, ldr, sig2);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Pivoted Cholesky (preconditioners.hpp:236-264), fp64, operation order of the
// reference: g = L[i,:s] . L[p,:s] (sequential), c_i -= g, L[i,s] = c_i / sqrt(d_p),
// d_i -= L[i,s]^2.  Each block also emits its (max d, lowest index) for the next pivot.
// ---------------------------------------------------------------------------
__global__ void pchol_step_kernel(double* __restrict__ L, long long ldl, int s, long long p, double root,
                                  const double* __restrict__ col, double* __restrict__ dg, int n,
                                  double* __restrict__ bval, long long* __restrict__ bidx) {
  extern __shared__ double lp[];  // L[p, 0..s)
  __shared__ double sv[kVT / 32];
  __shared__ long long si[kVT / 32];
  for (int c = threadIdx.x; c < s; c += blockDim.x) lp[c] = L[static_cast<long long>(c) * ldl + p];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double best = -DBL_MAX;
  long long bi = 0x7fffffffffffffffLL;
  if (i < n) {
    double g = 0.0;
    int c = 0;
    for (; c + 8 <= s; c += 8) {  // loads batched ahead of the (sequential, reference-order) sum
      double v8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v8[u] = L[static_cast<long long>(c + u) * ldl + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) g = __dadd_rn(g, __dmul_rn(v8[u], lp[c + u]));
    }
    for (; c < s; ++c) g = __dadd_rn(g, __dmul_rn(L[static_cast<long long>(c) * ldl + i], lp[c]));
    const double v = __ddiv_rn(__dsub_rn(col[i], g), root);
    L[static_cast<long long>(s) * ldl + i] = v;
    const double dn = __dsub_rn(dg[i], __dmul_rn(v, v));
    dg[i] = dn;
    best = dn;
    bi = i;
  }
  // (max, lowest index) block reduction
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sv[wid] = best;
    si[wid] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < blockDim.x / 32; ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
        best = sv[w];
        bi = si[w];
      }
    bval[blockIdx.x] = best;
    bidx[blockIdx.x] = bi;
  }
}

__global__ void argmax_finalize_kernel(const double* __restrict__ bval, const long long* __restrict__ bidx, int nb,
                                       double* __restrict__ out_val, long long* __restrict__ out_idx) {
  __shared__ double sv[kVT];
  __shared__ long long si[kVT];
  double best = -DBL_MAX;
  long long bi = 0x7fffffffffffffffLL;
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (bval[b] > best || (bval[b] == best && bidx[b] < bi)) {
      best = bval[b];
      bi = bidx[b];
    }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double ov = sv[threadIdx.x + o];
      const long long oi = si[threadIdx.x + o];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out_val = sv[0];
    *out_idx = si[0];
  }
}

// (max, lowest index) over an arbitrary vector (initial pivot).
__global__ void argmax_blocks_kernel(const double* __restrict__ v, int n, double* __restrict__ bval,
                                     long long* __restrict__ bidx) {
  __shared__ double sv[kVT];
  __shared__ long long si[kVT];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  sv[threadIdx.x] = i < n ? v[i] : -DBL_MAX;
  si[threadIdx.x] = i < n ? i : 0x7fffffffffffffffLL;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double ov = sv[threadIdx.x + o];
      const long long oi = si[threadIdx.x + o];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bval[blockIdx.x] = sv[0];
    bidx[blockIdx.x] = si[0];
  }
}

constexpr int kPB = 128;  // threads per pivoted-Cholesky step block (more CTAs per step)
int pchol_blocks(int n) { return (n + kPB - 1) / kPB; }

// ---------------------------------------------------------------------------
// Device-resident pivot state: the whole factorisation is enqueued without host
// round trips; a stopped state turns the remaining steps into no-ops.
// ---------------------------------------------------------------------------
cudaError_t launch_pchol_column_dev(int f, const double* sx, const double* sq, int n, int d, double o2,
                                    const PivotState* ps, double* out, cudaStream_t st);  // gpk_mvm.cu

__global__ void pchol_step_dev_kernel(double* __restrict__ L, long long ldl, int s, const double* __restrict__ col,
                                      double* __restrict__ dg, int n, const PivotState* __restrict__ ps,
                                      double* __restrict__ bval, long long* __restrict__ bidx) {
  extern __shared__ double lp[];
  __shared__ double sv[kVT / 32];
  __shared__ long long si[kVT / 32];
  if (ps->stopped) return;
  const long long p = ps->p;
  const double root = sqrt(ps->dp);  // preconditioners.hpp:256 (correctly rounded, as std::sqrt)
  for (int c = threadIdx.x; c < s; c += blockDim.x) lp[c] = L[static_cast<long long>(c) * ldl + p];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double best = -DBL_MAX;
  long long bi = 0x7fffffffffffffffLL;
  if (i < n) {
    double g = 0.0;
    int c = 0;
    for (; c + 8 <= s; c += 8) {  // loads batched ahead of the (sequential, reference-order) sum
      double v8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v8[u] = L[static_cast<long long>(c + u) * ldl + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) g = __dadd_rn(g, __dmul_rn(v8[u], lp[c + u]));
    }
    for (; c < s; ++c) g = __dadd_rn(g, __dmul_rn(L[static_cast<long long>(c) * ldl + i], lp[c]));
    const double v = __ddiv_rn(__dsub_rn(col[i], g), root);
    L[static_cast<long long>(s) * ldl + i] = v;
    const double dn = __dsub_rn(dg[i], __dmul_rn(v, v));
    dg[i] = dn;
    best = dn;
    bi = i;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sv[wid] = best;
    si[wid] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < blockDim.x / 32; ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
        best = sv[w];
        bi = si[w];
      }
    bval[blockIdx.x] = best;
    bidx[blockIdx.x] = bi;
  }
}

// next pivot (max remaining diagonal, lowest index on ties) and the stopping
// rules of preconditioners.hpp:250-253 for step s+1
__global__ void pchol_next_kernel(const double* __restrict__ bval, const long long* __restrict__ bidx, int nb, int s,
                                  double kmax, double diag_tol, PivotState* __restrict__ ps,
                                  long long* __restrict__ pivots) {
  __shared__ double sv[kVT];
  __shared__ long long si[kVT];
  if (ps->stopped) return;
  double best = -DBL_MAX;
  long long bi = 0x7fffffffffffffffLL;
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (bval[b] > best || (bval[b] == best && bidx[b] < bi)) {
      best = bval[b];
      bi = bidx[b];
    }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double ov = sv[threadIdx.x + o];
      const long long oi = si[threadIdx.x + o];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pivots[s] = ps->p;  // the pivot used at step s
    ps->dp = sv[0];
    ps->p = si[0];
    ps->done = s + 1;
    if (sv[0] < -1e-10 * kmax) {
      ps->stopped = 1;
      ps->negative = 1;
    } else if (sv[0] <= diag_tol) {
      ps->stopped = 1;
    }
  }
}

cudaError_t launch_pchol_dev(int family, const double* sx, const double* sq, int n, int d, double o2, double* L,
                             int rank, double diag_tol, double kmax, double* col, double* dg, double* bval,
                             long long* bidx, PivotState* ps, long long* pivots, cudaStream_t st) {
  const int nb = pchol_blocks(n);
  for (int s = 0; s < rank; ++s) {
    launch_pchol_column_dev(family, sx, sq, n, d, o2, ps, col, st);
    const size_t sm = sizeof(double) * static_cast<size_t>(s > 0 ? s : 1);
    pchol_step_dev_kernel<<<nb, kPB, sm, st>>>(L, n, s, col, dg, n, ps, bval, bidx);
    pchol_next_kernel<<<1, kVT, 0, st>>>(bval, bidx, nb, s, kmax, diag_tol, ps, pivots);
  }
  return cudaGetLastError();
}

cudaError_t launch_argmax(const double* v, int n, double* bval, long long* bidx, double* out_val,
                          long long* out_idx, cudaStream_t st) {
  const int nb = pchol_blocks(n);
  argmax_blocks_kernel<<<nb, kPB, 0, st>>>(v, n, bval, bidx);
  argmax_finalize_kernel<<<1, kVT, 0, st>>>(bval, bidx, nb, out_val, out_idx);
  return cudaGetLastError();
}

cudaError_t launch_pchol_step(double* L, long long ldl, int s, long long p, double root, const double* col, double* dg,
                              int n, double* bval, long long* bidx, double* out_val, long long* out_idx,
                              cudaStream_t st) {
  const int nb = pchol_blocks(n);
  const size_t sm = sizeof(double) * static_cast<size_t>(s > 0 ? s : 1);
  pchol_step_kernel<<<nb, kPB, sm, st>>>(L, ldl, s, p, root, col, dg, n, bval, bidx);
  argmax_finalize_kernel<<<1, kVT, 0, st>>>(bval, bidx, nb, out_val, out_idx);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Frozen-pivot derivative factors (preconditioners.hpp:278-293), batched over
// the non-noise parameters (blockIdx.y = w):
//   dc = dKcol_w - dL_w[:, :s] L[p, :s]' - L[:, :s] dL_w[p, :s]'
//   dL_w[:, s] = dc / L[p,s] - L[:, s] * (dc[p] / (2 L[p,s] L[p,s]))
// ---------------------------------------------------------------------------
__global__ void dl_step_kernel(const double* __restrict__ L, long long ldl, double* __restrict__ dL, long long wstride,
                               int s, long long p, const double* __restrict__ dcol, long long dcol_stride, int n) {
  extern __shared__ double sh[];  // [0,s): L[p,:s]; [s,2s): dL_w[p,:s]
  __shared__ double dd_sh;
  const int w = blockIdx.y;
  double* dLw = dL + w * wstride;
  const double* dcw = dcol + w * dcol_stride;
  for (int c = threadIdx.x; c < s; c += blockDim.x) {
    sh[c] = L[static_cast<long long>(c) * ldl + p];
    sh[s + c] = dLw[static_cast<long long>(c) * ldl + p];
  }
  __syncthreads();
  auto dc_at = [&](long long i) {
    double g1 = 0.0, g2 = 0.0;
    for (int c = 0; c < s; ++c) g1 = __dadd_rn(g1, __dmul_rn(dLw[static_cast<long long>(c) * ldl + i], sh[c]));
    for (int c = 0; c < s; ++c) g2 = __dadd_rn(g2, __dmul_rn(L[static_cast<long long>(c) * ldl + i], sh[s + c]));
    return __dsub_rn(__dsub_rn(dcw[i], g1), g2);
  };
  if (threadIdx.x == 0) dd_sh = dc_at(p);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double root = L[static_cast<long long>(s) * ldl + p];
  const double dc = dc_at(i);
  const double corr = __ddiv_rn(dd_sh, __dmul_rn(__dmul_rn(2.0, root), root));
  dLw[static_cast<long long>(s) * ldl + i] =
      __dsub_rn(__ddiv_rn(dc, root), __dmul_rn(L[static_cast<long long>(s) * ldl + i], corr));
}

// Blocked variant (columns s0..s0+b-1 after the block update DC_w -= dL_w[:, :s0] Lp + L[:, :s0] dLp_w was
// applied by GEMMs): in-block step for column j = s0 + q of every parameter w (blockIdx.y):
//   dc = DC_w[:, q] - dL_w[:, s0:j] L[p, s0:j]' - L[:, s0:j] dL_w[p, s0:j]'
//   dL_w[:, j] = dc / L[p,j] - L[:, j] * (dc[p] / (2 L[p,j] L[p,j]))
// dc[p] is recomputed per CTA with the same operation order as row p's own value.
__global__ void dl_inblock_kernel(const double* __restrict__ L, long long ldl, double* __restrict__ dL,
                                  long long wstride, int s0, int q, long long p, const double* __restrict__ DC,
                                  long long dcw_stride, int n) {
  __shared__ double lp[64], dlp[64];
  __shared__ double dd_sh;
  const int w = blockIdx.y;
  double* dLw = dL + w * wstride;
  const double* dcw = DC + w * dcw_stride + static_cast<long long>(q) * ldl;
  for (int c = threadIdx.x; c < q; c += blockDim.x) {
    lp[c] = L[static_cast<long long>(s0 + c) * ldl + p];
    dlp[c] = dLw[static_cast<long long>(s0 + c) * ldl + p];
  }
  __syncthreads();
  auto dc_at = [&](long long i) {
    double g1 = 0.0, g2 = 0.0;
    for (int c = 0; c < q; ++c) g1 = __dadd_rn(g1, __dmul_rn(dLw[static_cast<long long>(s0 + c) * ldl + i], lp[c]));
    for (int c = 0; c < q; ++c) g2 = __dadd_rn(g2, __dmul_rn(L[static_cast<long long>(s0 + c) * ldl + i], dlp[c]));
    return __dsub_rn(__dsub_rn(dcw[i], g1), g2);
  };
  if (threadIdx.x == 0) {  // row p's value from the staged pivot rows (same operation order)
    double g1 = 0.0, g2 = 0.0;
    for (int c = 0; c < q; ++c) g1 = __dadd_rn(g1, __dmul_rn(dlp[c], lp[c]));
    for (int c = 0; c < q; ++c) g2 = __dadd_rn(g2, __dmul_rn(lp[c], dlp[c]));
    dd_sh = __dsub_rn(__dsub_rn(dcw[p], g1), g2);
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = s0 + q;
  const double root = L[static_cast<long long>(j) * ldl + p];
  const double dc = dc_at(i);
  const double corr = __ddiv_rn(dd_sh, __dmul_rn(__dmul_rn(2.0, root), root));
  dLw[static_cast<long long>(j) * ldl + i] =
      __dsub_rn(__ddiv_rn(dc, root), __dmul_rn(L[static_cast<long long>(j) * ldl + i], corr));
}

cudaError_t launch_dl_inblock(const double* L, long long ldl, double* dL, long long wstride, int nw, int s0, int q,
                              long long p, const double* DC, long long dcw_stride, int n, cudaStream_t st) {
  dim3 g(pchol_blocks(n), nw);
  dl_inblock_kernel<<<g, kPB, 0, st>>>(L, ldl, dL, wstride, s0, q, p, DC, dcw_stride, n);
  return cudaGetLastError();
}

// out[w][q][c] = M_w[piv[q], c] for c < s0  (column-major s0 x b blocks, one per w; wstride 0 => single)
__global__ void gather_pivot_rows_kernel(const double* __restrict__ M, long long ldm, long long mstride,
                                         const long long* __restrict__ piv, int s0, int b,
                                         double* __restrict__ out) {
  const int w = blockIdx.y;
  const long long tot = static_cast<long long>(s0) * b;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e % s0), q = static_cast<int>(e / s0);
    out[w * tot + e] = M[w * mstride + static_cast<long long>(c) * ldm + piv[q]];
  }
}

cudaError_t launch_gather_pivot_rows(const double* M, long long ldm, long long mstride, int nw,
                                     const long long* piv, int s0, int b, double* out, cudaStream_t st) {
  const long long tot = static_cast<long long>(s0) * b;
  dim3 g(static_cast<unsigned>(std::min<long long>((tot + kVT - 1) / kVT, 1024)), nw);
  gather_pivot_rows_kernel<<<g, kVT, 0, st>>>(M, ldm, mstride, piv, s0, b, out);
  return cudaGetLastError();
}

cudaError_t launch_dl_step(const double* L, long long ldl, double* dL, long long wstride, int nw, int s, long long p,
                           const double* dcol, long long dcol_stride, int n, cudaStream_t st) {
  dim3 g(pchol_blocks(n), nw);
  const size_t sm = sizeof(double) * static_cast<size_t>(2 * (s > 0 ? s : 1));
  dl_step_kernel<<<g, kPB, sm, st>>>(L, ldl, dL, wstride, s, p, dcol, dcol_stride, n);
  return cudaGetLastError();
}

}  // namespace gpk
