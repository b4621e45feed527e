// Persistent pivoted Cholesky and blocked frozen-pivot derivative factors (fp64).
//
// pchol_persistent_kernel: the whole greedy factorisation of
// preconditioners.hpp:236-264 in ONE cooperative launch.  Per step every CTA
// evaluates the pivot's kernel column for its rows (kernels.hpp:235-243 operation
// order), the Schur update c -= L[:, :s] L[p, :s]' (sequential sum, reference
// order), L[:, s] = c / sqrt(d_p), d -= L[:, s]^2, and its (max d, lowest index)
// candidate; after one grid barrier every CTA reduces all candidates itself, so
// the CTAs agree on the next pivot without a second barrier (candidates are
// double-buffered by step parity).  The arithmetic per row is the one of the
// per-step kernels it replaces (pchol_column_dev / pchol_step_dev / pchol_next in
// gpk_mvm.cu, gpk_linalg.cu): same pivots, bitwise the same L.
//
// deriv_columns_block / dl_replay / dl_block: preconditioners.hpp:278-293 for a
// block of kDB pivots in three launches (instead of two per column): the dK columns
// of all pivots of the block at once; the in-block recursion restricted to the
// block's own pivot rows (bb x bb per parameter, one small CTA each), which is all
// that couples the rows; then every row runs all bb columns from registers.  Same
// operation order as dl_inblock_kernel (bitwise the same dL).
#include <cooperative_groups.h>

#include <cfloat>
#include <climits>

#include "gpk_common.cuh"
#include "gpk_internal.h"
#include "gpk_linalg.h"
#include "gpk_ref_shape.cuh"

namespace cg = cooperative_groups;

namespace gpk {

constexpr int kPT = 128;  // threads per CTA
constexpr int kDB = 32;   // derivative-factor block (columns)

GPK_DEV void better(double& bv, long long& bi, double ov, long long oi) {
  if (ov > bv || (ov == bv && oi < bi)) {
    bv = ov;
    bi = oi;
  }
}

// (max, lowest index) over the CTA; result valid in every thread
GPK_DEV void block_best(double& bv, long long& bi, double* sv, long long* si) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();  // sv / si reuse across calls
  if (lane == 0) {
    sv[wid] = bv;
    si[wid] = bi;
  }
  __syncthreads();
  bv = sv[0];
  bi = si[0];
  for (int w = 1; w < kPT / 32; ++w) better(bv, bi, sv[w], si[w]);
}

__global__ void __launch_bounds__(kPT) pchol_persistent_kernel(int f, const double* __restrict__ sx,
                                                               const double* __restrict__ sq, int n, int d, double o2,
                                                               double* __restrict__ L, int rank, double diag_tol,
                                                               double kmax, double* __restrict__ dg,
                                                               double* __restrict__ cval, long long* __restrict__ cidx,
                                                               PivotState* __restrict__ ps,
                                                               long long* __restrict__ pivots) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double lp[];  // L[p, 0..s)
  __shared__ double xp[32];
  __shared__ double sv[kPT / 32];
  __shared__ long long si[kPT / 32];
  const int G = gridDim.x;
  double dp = ps->dp;
  long long p = ps->p;
  for (int s = 0; s < rank; ++s) {
    const double root = sqrt(dp);  // preconditioners.hpp:256 (correctly rounded, as std::sqrt)
    for (int c = threadIdx.x; c < s; c += kPT) lp[c] = L[static_cast<long long>(c) * n + p];
    for (int k = threadIdx.x; k < d; k += kPT) xp[k] = sx[static_cast<long long>(k) * n + p];
    __syncthreads();
    const double sqp = sq[p];
    double best = -DBL_MAX;
    long long bi = LLONG_MAX;
    for (int i = blockIdx.x * kPT + threadIdx.x; i < n; i += G * kPT) {
      // kernel column (kernels.hpp:235-243)
      double g = 0.0;
      for (int k = 0; k < d; ++k) g = __dadd_rn(g, __dmul_rn(sx[static_cast<long long>(k) * n + i], xp[k]));
      double sd = __dsub_rn(__dadd_rn(sq[i], sqp), __dmul_rn(2.0, g));
      sd = sd > 0.0 ? sd : 0.0;
      const double col = __dmul_rn(o2, ref_shape(f, sd));
      // Schur update, sequential reference-order sum (loads batched ahead of the adds)
      double h = 0.0;
      int c = 0;
      for (; c + 8 <= s; c += 8) {
        double v8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v8[u] = L[static_cast<long long>(c + u) * n + i];
#pragma unroll
        for (int u = 0; u < 8; ++u) h = __dadd_rn(h, __dmul_rn(v8[u], lp[c + u]));
      }
      for (; c < s; ++c) h = __dadd_rn(h, __dmul_rn(L[static_cast<long long>(c) * n + i], lp[c]));
      const double v = __ddiv_rn(__dsub_rn(col, h), root);
      L[static_cast<long long>(s) * n + i] = v;
      const double dn = __dsub_rn(dg[i], __dmul_rn(v, v));
      dg[i] = dn;
      better(best, bi, dn, i);
    }
    block_best(best, bi, sv, si);
    const int par = (s & 1) * G;
    if (threadIdx.x == 0) {
      cval[par + blockIdx.x] = best;
      cidx[par + blockIdx.x] = bi;
    }
    grid.sync();
    double nv = -DBL_MAX;
    long long ni = LLONG_MAX;
    for (int b = threadIdx.x; b < G; b += kPT) better(nv, ni, cval[par + b], cidx[par + b]);
    block_best(nv, ni, sv, si);
    const bool negative = nv < -1e-10 * kmax;  // :250-252
    const bool stop = negative || nv <= diag_tol;  // :253
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      pivots[s] = p;
      ps->dp = nv;
      ps->p = ni;
      ps->done = s + 1;
      ps->stopped = stop ? 1 : 0;
      ps->negative = negative ? 1 : 0;
    }
    dp = nv;
    p = ni;
    if (stop) break;
    __syncthreads();  // lp / xp of this step fully consumed
  }
}

int pchol_persistent_grid(int n, size_t smem) {
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, pchol_persistent_kernel, kPT, smem) != cudaSuccess)
    return 0;
  const long long need = (static_cast<long long>(n) + kPT - 1) / kPT;
  const long long cap = static_cast<long long>(per) * sms;
  return static_cast<int>(need < cap ? need : cap);
}

cudaError_t launch_pchol_persistent(int family, const double* sx, const double* sq, int n, int d, double o2,
                                    double* L, int rank, double diag_tol, double kmax, double* dg, double* cval,
                                    long long* cidx, PivotState* ps, long long* pivots, int grid, cudaStream_t st) {
  const size_t smem = sizeof(double) * static_cast<size_t>(rank > 0 ? rank : 1);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(pchol_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  void* args[] = {&family, &sx, &sq, &n, &d, &o2, &L, &rank, &diag_tol, &kmax, &dg, &cval, &cidx, &ps, &pivots};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(pchol_persistent_kernel), dim3(grid), dim3(kPT),
                                     args, smem, st);
}

// ---------------------------------------------------------------------------
// Frozen-pivot derivative factors, one block of bb <= kDB pivots (s0 .. s0+bb-1).
// ---------------------------------------------------------------------------
// DC_w[q][i] = dK_w column of pivot piv[q] (kernels.hpp:252-267), blockIdx.y = q
__global__ void deriv_columns_block_kernel(int f, const double* __restrict__ sx, const double* __restrict__ x,
                                           const double* __restrict__ sq, int n, int d,
                                           const long long* __restrict__ piv, int nw,
                                           const double* __restrict__ facs, double o2, double* __restrict__ DC,
                                           long long dcw_stride) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int q = blockIdx.y;
  const long long p = piv[q];
  double g = 0.0;
  for (int k = 0; k < d; ++k) g = __dadd_rn(g, __dmul_rn(sx[static_cast<long long>(k) * n + r], sx[k * n + p]));
  double s = __dsub_rn(__dadd_rn(sq[r], sq[p]), __dmul_rn(2.0, g));
  s = s > 0.0 ? s : 0.0;
  double* out = DC + static_cast<long long>(q) * n + r;
  out[0] = __dmul_rn(facs[0], __dmul_rn(o2, ref_shape(f, s)));
  if (nw > 1) {
    const double ds = ref_shape_ds(f, s);
    for (int w = 1; w < nw; ++w) {
      const int j = w - 1;
      const double dx = __dsub_rn(x[static_cast<long long>(j) * n + r], x[static_cast<long long>(j) * n + p]);
      out[w * dcw_stride] = __dmul_rn(facs[w], __dmul_rn(ds, __dmul_rn(dx, dx)));
    }
  }
}

cudaError_t launch_deriv_columns_block(int family, const double* sx, const double* x, const double* sq, int n, int d,
                                       const long long* piv, int bb, int nw, const double* facs, double o2,
                                       double* DC, long long dcw_stride, cudaStream_t st) {
  dim3 g((n + 127) / 128, bb);
  deriv_columns_block_kernel<<<g, 128, 0, st>>>(family, sx, x, sq, n, d, piv, nw, facs, o2, DC, dcw_stride);
  return cudaGetLastError();
}

// In-block recursion for columns j = s0 + q, q < bb, of parameter w, after the block
// update DC_w -= dL_w[:, :s0] Lp + L[:, :s0] dLp_w:
//   dc_i = (DC_w[i, q] - sum_{c<q} dL_w[i, s0+c] L[p_j, s0+c]) - sum_{c<q} L[i, s0+c] dL_w[p_j, s0+c]
//   dL_w[i, j] = dc_i / L[p_j, j] - L[i, j] * (dc_{p_j} / (2 L[p_j, j] L[p_j, j]))
// Step 1 (dl_replay_kernel, one CTA per w): the recursion on the block's own pivot rows,
// rep_w = {Lpp[q'][c], Dp[q'][c], root[q], corr[q]}; step 2 (dl_block_kernel): every row.
constexpr int kRep = 2 * kDB * kDB + 2 * kDB;  // doubles per parameter in the replay buffer

__global__ void dl_replay_kernel(const double* __restrict__ L, int s0, int bb, const long long* __restrict__ piv,
                                 const double* __restrict__ DC, long long dcw_stride, int n,
                                 double* __restrict__ rep) {
  __shared__ double Lpp[kDB][kDB + 1], Dp[kDB][kDB + 1], dcq[kDB];
  __shared__ double rootq[kDB], corrq[kDB];
  const int w = blockIdx.x;
  const double* DCw = DC + w * dcw_stride;
  const int qq = threadIdx.x;  // one thread per pivot row of the block
  for (int e = threadIdx.x; e < bb * bb; e += blockDim.x) {
    const int a = e / bb, c = e % bb;
    Lpp[a][c] = L[static_cast<long long>(s0 + c) * n + piv[a]];
  }
  __syncthreads();
  for (int q = 0; q < bb; ++q) {
    double dc = 0.0;
    if (qq < bb) {  // row p_qq at column q (row p_q's value is dc_{p_q})
      double g1 = 0.0, g2 = 0.0;
      for (int c = 0; c < q; ++c) g1 = __dadd_rn(g1, __dmul_rn(Dp[qq][c], Lpp[q][c]));
      for (int c = 0; c < q; ++c) g2 = __dadd_rn(g2, __dmul_rn(Lpp[qq][c], Dp[q][c]));
      dc = __dsub_rn(__dsub_rn(DCw[static_cast<long long>(q) * n + piv[qq]], g1), g2);
      if (qq == q) {
        const double root = Lpp[q][q];
        rootq[q] = root;
        corrq[q] = __ddiv_rn(dc, __dmul_rn(__dmul_rn(2.0, root), root));
      }
    }
    __syncthreads();
    if (qq < bb) Dp[qq][q] = __dsub_rn(__ddiv_rn(dc, rootq[q]), __dmul_rn(Lpp[qq][q], corrq[q]));
    __syncthreads();
  }
  double* r = rep + static_cast<long long>(w) * kRep;
  for (int e = threadIdx.x; e < kDB * kDB; e += blockDim.x) {
    const int a = e / kDB, c = e % kDB;
    r[e] = (a < bb && c < bb) ? Lpp[a][c] : 0.0;
    r[kDB * kDB + e] = (a < bb && c < bb) ? Dp[a][c] : 0.0;
  }
  if (threadIdx.x < kDB) {
    r[2 * kDB * kDB + threadIdx.x] = threadIdx.x < bb ? rootq[threadIdx.x] : 1.0;
    r[2 * kDB * kDB + kDB + threadIdx.x] = threadIdx.x < bb ? corrq[threadIdx.x] : 0.0;
  }
}

__global__ void __launch_bounds__(kPT) dl_block_kernel(const double* __restrict__ L, double* __restrict__ dL,
                                                       long long wstride, int s0, int bb,
                                                       const double* __restrict__ DC, long long dcw_stride, int n,
                                                       const double* __restrict__ rep) {
  __shared__ double Lpp[kDB][kDB], Dp[kDB][kDB], rootq[kDB], corrq[kDB];
  const int w = blockIdx.y;
  double* dLw = dL + w * wstride;
  const double* DCw = DC + w * dcw_stride;
  const double* r = rep + static_cast<long long>(w) * kRep;
  for (int e = threadIdx.x; e < kDB * kDB; e += kPT) {
    (&Lpp[0][0])[e] = r[e];
    (&Dp[0][0])[e] = r[kDB * kDB + e];
  }
  if (threadIdx.x < kDB) {
    rootq[threadIdx.x] = r[2 * kDB * kDB + threadIdx.x];
    corrq[threadIdx.x] = r[2 * kDB * kDB + kDB + threadIdx.x];
  }
  __syncthreads();
  for (int i = blockIdx.x * kPT + threadIdx.x; i < n; i += gridDim.x * kPT) {
    double li[kDB], dli[kDB];
#pragma unroll
    for (int c = 0; c < kDB; ++c) li[c] = c < bb ? L[static_cast<long long>(s0 + c) * n + i] : 0.0;
#pragma unroll
    for (int q = 0; q < kDB; ++q) {
      if (q < bb) {
        double g1 = 0.0, g2 = 0.0;
#pragma unroll
        for (int c = 0; c < q; ++c) g1 = __dadd_rn(g1, __dmul_rn(dli[c], Lpp[q][c]));
#pragma unroll
        for (int c = 0; c < q; ++c) g2 = __dadd_rn(g2, __dmul_rn(li[c], Dp[q][c]));
        const double dc = __dsub_rn(__dsub_rn(DCw[static_cast<long long>(q) * n + i], g1), g2);
        dli[q] = __dsub_rn(__ddiv_rn(dc, rootq[q]), __dmul_rn(li[q], corrq[q]));
        dLw[static_cast<long long>(s0 + q) * n + i] = dli[q];
      }
    }
  }
}

size_t dl_replay_workspace(int nw) { return static_cast<size_t>(nw) * kRep; }

cudaError_t launch_dl_block(const double* L, double* dL, long long wstride, int nw, int s0, int bb,
                            const long long* piv, const double* DC, long long dcw_stride, int n, double* rep,
                            cudaStream_t st) {
  if (bb < 1 || bb > kDB) return cudaErrorInvalidValue;
  dl_replay_kernel<<<nw, kDB, 0, st>>>(L, s0, bb, piv, DC, dcw_stride, n, rep);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int need = (n + kPT - 1) / kPT;
  const int gx = need < 4 * sms ? need : 4 * sms;
  dim3 g(gx > 0 ? gx : 1, nw);
  dl_block_kernel<<<g, kPT, 0, st>>>(L, dL, wstride, s0, bb, DC, dcw_stride, n, rep);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Row-sharded pivoted Cholesky (world > 1): every rank owns the rows
// [r0, r0 + nl) of L (local leading dimension ldl) and of the diagonal.  Per step, all
// stream-ordered (no host round trip; a fired stopping rule turns later steps into no-ops):
//   pchol_shard_step : column s on the own rows -- exactly pchol_persistent_kernel's per-row
//                      arithmetic, so the rows and the diagonal are bitwise the unsharded
//                      ones -- and per-CTA (max, lowest index) candidates
//   pchol_shard_best : the rank's candidate (max, lowest GLOBAL index)
//   [all-gather of the world's candidates]
//   pchol_shard_select: the global pivot (max, lowest index over ranks in rank order =
//                      index order: the reference's strict '>' scan, preconditioners.hpp:
//                      247-249) and the stopping rules (:250-253)
//   pchol_shard_rowpack: the owner of the new pivot p sends L[p, 0..s]
//   [all-gather]  pchol_shard_rowtake: every rank takes the owner's row as the next L[p, :s]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kPT) pchol_shard_step_kernel(int f, const double* __restrict__ sx,
                                                               const double* __restrict__ sq, int n, int d,
                                                               double o2, double* __restrict__ L, long long ldl,
                                                               int r0, int nl, int s, const double* __restrict__ lpg,
                                                               const PivotState* __restrict__ ps,
                                                               double* __restrict__ dg, double* __restrict__ cval,
                                                               long long* __restrict__ cidx) {
  extern __shared__ double lp[];
  __shared__ double xp[32];
  __shared__ double sv[kPT / 32];
  __shared__ long long si[kPT / 32];
  if (ps->stopped) return;
  const long long p = ps->p;
  const double root = sqrt(ps->dp);  // preconditioners.hpp:256
  for (int c = threadIdx.x; c < s; c += kPT) lp[c] = lpg[c];
  for (int k = threadIdx.x; k < d; k += kPT) xp[k] = sx[static_cast<long long>(k) * n + p];
  __syncthreads();
  const double sqp = sq[p];
  double best = -DBL_MAX;
  long long bi = LLONG_MAX;
  for (int j = blockIdx.x * kPT + threadIdx.x; j < nl; j += gridDim.x * kPT) {
    const long long i = r0 + j;
    double g = 0.0;
    for (int k = 0; k < d; ++k) g = __dadd_rn(g, __dmul_rn(sx[static_cast<long long>(k) * n + i], xp[k]));
    double sd = __dsub_rn(__dadd_rn(sq[i], sqp), __dmul_rn(2.0, g));
    sd = sd > 0.0 ? sd : 0.0;
    const double col = __dmul_rn(o2, ref_shape(f, sd));
    double h = 0.0;
    int c = 0;
    for (; c + 8 <= s; c += 8) {
      double v8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v8[u] = L[static_cast<long long>(c + u) * ldl + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) h = __dadd_rn(h, __dmul_rn(v8[u], lp[c + u]));
    }
    for (; c < s; ++c) h = __dadd_rn(h, __dmul_rn(L[static_cast<long long>(c) * ldl + j], lp[c]));
    const double v = __ddiv_rn(__dsub_rn(col, h), root);
    L[static_cast<long long>(s) * ldl + j] = v;
    const double dn = __dsub_rn(dg[j], __dmul_rn(v, v));
    dg[j] = dn;
    better(best, bi, dn, i);
  }
  block_best(best, bi, sv, si);
  if (threadIdx.x == 0) {
    cval[blockIdx.x] = best;
    cidx[blockIdx.x] = bi;
  }
}

// the rank's candidate over the G CTA candidates -> send = {value, index as double bits}
__global__ void __launch_bounds__(kPT) pchol_shard_best_kernel(const double* __restrict__ cval,
                                                               const long long* __restrict__ cidx, int G,
                                                               const PivotState* __restrict__ ps,
                                                               double* __restrict__ send) {
  __shared__ double sv[kPT / 32];
  __shared__ long long si[kPT / 32];
  if (ps->stopped) return;
  double bv = -DBL_MAX;
  long long bi = LLONG_MAX;
  for (int b = threadIdx.x; b < G; b += kPT) better(bv, bi, cval[b], cidx[b]);
  block_best(bv, bi, sv, si);
  if (threadIdx.x == 0) {
    send[0] = bv;
    send[1] = __longlong_as_double(bi);
  }
}

// global pivot over the world's candidates (rank order), stopping rules, pivot record
__global__ void pchol_shard_select_kernel(const double* __restrict__ cand, int world, int s, double diag_tol,
                                          double kmax, PivotState* __restrict__ ps, long long* __restrict__ pivots) {
  if (threadIdx.x != 0 || ps->stopped) return;
  double nv = -DBL_MAX;
  long long ni = LLONG_MAX;
  for (int r = 0; r < world; ++r) better(nv, ni, cand[2 * r], __double_as_longlong(cand[2 * r + 1]));
  const bool negative = nv < -1e-10 * kmax;      // :250-252
  const bool stop = negative || nv <= diag_tol;  // :253
  pivots[s] = ps->p;
  ps->dp = nv;
  ps->p = ni;
  ps->done = s + 1;
  ps->stopped = stop ? 1 : 0;
  ps->negative = negative ? 1 : 0;
}

// the owner of the (new) pivot packs L[p, 0..s] (k doubles, zero beyond s and on other ranks)
__global__ void pchol_shard_rowpack_kernel(const double* __restrict__ L, long long ldl, int r0, int nl, int s, int k,
                                           const PivotState* __restrict__ ps, double* __restrict__ send) {
  const long long p = ps->p;
  const bool mine = !ps->stopped && p >= r0 && p < r0 + nl;
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    send[c] = (mine && c <= s) ? L[static_cast<long long>(c) * ldl + (p - r0)] : 0.0;
}

// every rank takes the owner's row: lp[c] = recv[owner][c]
__global__ void pchol_shard_rowtake_kernel(const double* __restrict__ recv, int world, int k,
                                           const int* __restrict__ rr0, const int* __restrict__ rrows,
                                           const PivotState* __restrict__ ps, double* __restrict__ lp) {
  if (ps->stopped) return;
  const long long p = ps->p;
  int owner = 0;
  for (int r = 0; r < world; ++r)
    if (p >= rr0[r] && p < rr0[r] + rrows[r]) owner = r;
  for (int c = threadIdx.x; c < k; c += blockDim.x) lp[c] = recv[static_cast<long long>(owner) * k + c];
}

// rows of pivots owned by this rank -> send[q][c] (k x k, zero for other ranks' pivots)
__global__ void pchol_pivot_rows_pack_kernel(const double* __restrict__ L, long long ldl, int r0, int nl, int k,
                                             const long long* __restrict__ piv, double* __restrict__ send) {
  const int q = blockIdx.x;
  const long long p = piv[q];
  const bool mine = p >= r0 && p < r0 + nl;
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    send[static_cast<long long>(q) * k + c] = mine ? L[static_cast<long long>(c) * ldl + (p - r0)] : 0.0;
}

// L[nl + q, c] = the owner's row of pivot q (the extended rows of the sharded factor)
__global__ void pchol_pivot_rows_take_kernel(const double* __restrict__ recv, int world, int k,
                                             const int* __restrict__ rr0, const int* __restrict__ rrows,
                                             const long long* __restrict__ piv, double* __restrict__ L,
                                             long long ldl, int nl) {
  const int q = blockIdx.x;
  const long long p = piv[q];
  int owner = 0;
  for (int r = 0; r < world; ++r)
    if (p >= rr0[r] && p < rr0[r] + rrows[r]) owner = r;
  const double* src = recv + (static_cast<long long>(owner) * k + q) * k;
  for (int c = threadIdx.x; c < k; c += blockDim.x) L[static_cast<long long>(c) * ldl + nl + q] = src[c];
}

int pchol_shard_grid(int nl) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int need = (nl + kPT - 1) / kPT;
  return need < 4 * sms ? (need > 0 ? need : 1) : 4 * sms;
}

cudaError_t launch_pchol_shard_step(int family, const double* sx, const double* sq, int n, int d, double o2,
                                    double* L, long long ldl, int r0, int nl, int s, const double* lp,
                                    const PivotState* ps, double* dg, double* cval, long long* cidx, int grid,
                                    double* send, cudaStream_t st) {
  const size_t smem = sizeof(double) * static_cast<size_t>(s > 0 ? s : 1);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(pchol_shard_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  pchol_shard_step_kernel<<<grid, kPT, smem, st>>>(family, sx, sq, n, d, o2, L, ldl, r0, nl, s, lp, ps, dg, cval,
                                                   cidx);
  pchol_shard_best_kernel<<<1, kPT, 0, st>>>(cval, cidx, grid, ps, send);
  return cudaGetLastError();
}

cudaError_t launch_pchol_shard_select(const double* cand, int world, int s, double diag_tol, double kmax,
                                      PivotState* ps, long long* pivots, const double* L, long long ldl, int r0,
                                      int nl, int k, double* rowsend, cudaStream_t st) {
  pchol_shard_select_kernel<<<1, 32, 0, st>>>(cand, world, s, diag_tol, kmax, ps, pivots);
  pchol_shard_rowpack_kernel<<<1, 256, 0, st>>>(L, ldl, r0, nl, s, k, ps, rowsend);
  return cudaGetLastError();
}

cudaError_t launch_pchol_shard_rowtake(const double* recv, int world, int k, const int* rr0, const int* rrows,
                                       const PivotState* ps, double* lp, cudaStream_t st) {
  pchol_shard_rowtake_kernel<<<1, 256, 0, st>>>(recv, world, k, rr0, rrows, ps, lp);
  return cudaGetLastError();
}

cudaError_t launch_pchol_pivot_rows(int phase, const double* src, double* dst, long long ldl, int r0, int nl, int k,
                                    const long long* piv, int world, const int* rr0, const int* rrows,
                                    cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  if (phase == 0)
    pchol_pivot_rows_pack_kernel<<<k, 128, 0, st>>>(src, ldl, r0, nl, k, piv, dst);
  else
    pchol_pivot_rows_take_kernel<<<k, 128, 0, st>>>(src, world, k, rr0, rrows, piv, dst, ldl, nl);
  return cudaGetLastError();
}

// extended coordinate rows for the sharded derivative factors: rows [0, nl) = global rows
// r0 .. r0 + nl - 1, rows [nl, nl + k) = the pivots (column-major, leading dimension ne)
__global__ void gather_ext_rows_kernel(const double* __restrict__ src, long long lds, int cols, int r0, int nl,
                                       const long long* __restrict__ piv, int k, double* __restrict__ dst,
                                       long long ne) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= nl + k || c >= cols) return;
  const long long g = i < nl ? r0 + i : piv[i - nl];
  dst[c * ne + i] = src[c * lds + g];
}

cudaError_t launch_gather_ext_rows(const double* src, long long lds, int cols, int r0, int nl, const long long* piv,
                                   int k, double* dst, long long ne, cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  dim3 g(static_cast<unsigned>((nl + k + 255) / 256), cols);
  gather_ext_rows_kernel<<<g, 256, 0, st>>>(src, lds, cols, r0, nl, piv, k, dst, ne);
  return cudaGetLastError();
}

// piv_ext[q] = nl + q
__global__ void iota_ll_kernel(long long* __restrict__ out, int k, long long base) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < k) out[q] = base + q;
}
cudaError_t launch_iota_ll(long long* out, int k, long long base, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  iota_ll_kernel<<<(k + 255) / 256, 256, 0, st>>>(out, k, base);
  return cudaGetLastError();
}

}  // namespace gpk
