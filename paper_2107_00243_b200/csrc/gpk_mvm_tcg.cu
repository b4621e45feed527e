// Front end of the Gram-variant tensor-core MVM (gpk_mvm_tcg.cuh): packing of
// the centred, pre-scaled coordinates into tf32 hi/lo 128B-swizzled K-major
// tiles plus their fp32 squared norms, and dispatch.
#include <algorithm>

#include "gpk_mvm_tcg.cuh"

namespace gpk {
namespace tcg {
template <int FAM>
cudaError_t launch_tcg_fam(int ks, int dpd, int nc8, const float* Xh, const float* Xl, const float* Xn,
                           const float* X32, const __half* Vhi, const __half* Vlo, const double* colscale,
                           double* out, const MvmArgs& a, dim3 g, cudaStream_t st);
}

// mu[k] = mean_i X[i, k] / l_k (fixed-order block reduction, one block per coordinate)
__global__ void gram_mean_kernel(const double* __restrict__ X, long long ldx, int n, const double* __restrict__ ls,
                                 double* __restrict__ mu) {
  __shared__ double red[256];
  const int k = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += X[k * ldx + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) mu[k] = red[0] / n / ls[k];
}

// one thread per row: x~ = (X/l - mu) sqrt(prescale), n = |x~|^2 (fp32), and the two
// AUGMENTED coordinate images of the Gram MMA, split into tf32 hi / lo at the swizzled
// positions of the tile image (padded rows / coordinates zero):
//   B side (the j-tiles, xh / xl):              [ x~ (d) , 1 , n ]
//   A side (the row operand, xh / xl + 32 n_pad): [ -2 x~ (d), n , 1 ]
// so that A_i . B_j = n_i + n_j - 2 x~_i . x~_j = s_ij comes out of the tensor cores directly
// (the -2 is exact in the split; n and 1 split into hi + lo like every coordinate).  xn[i] = n;
// xn[n_pad + jt] = max over j-tile jt of n (the per-tile bound of the cancellation guard).
__global__ void gram_pack_kernel(const double* __restrict__ X, long long ldx, int n, int d, int n_pad,
                                 const double* __restrict__ ls, const double* __restrict__ mu, double pre,
                                 float* __restrict__ xh, float* __restrict__ xl, float* __restrict__ xn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  const long long tile = i >> 5;
  const int r = i & 31;
  const bool real = i < n;
  float nrm = 0.0f;
  for (int k = 0; k < d; ++k) {
    const float v = real ? static_cast<float>((X[k * ldx + i] / ls[k] - mu[k]) * pre) : 0.0f;
    nrm = fmaf(v, v, nrm);
  }
  const long long aoff = static_cast<long long>(n_pad) * 32;
  for (int k = 0; k < 32; ++k) {
    // padded rows keep their 1 entries (with x~ = 0, n = 0): s(real i, padded j) = |x_i|^2 and
    // s(padded i, real j) = |x_j|^2 as in the non-augmented form, never "near pairs" -- an
    // all-zero image would make every entry of a padded row block a guard-path entry
    float vb = 0.0f, va = 0.0f;
    if (k < d) {
      vb = real ? static_cast<float>((X[k * ldx + i] / ls[k] - mu[k]) * pre) : 0.0f;
      va = -2.0f * vb;
    } else if (k == d) {
      vb = 1.0f;
      va = nrm;
    } else if (k == d + 1) {
      vb = nrm;
      va = 1.0f;
    }
    const long long off = tile * 1024 + ((r >> 3) * 256 + (r & 7) * 32 + ((((k >> 2) ^ (r & 7))) << 2) + (k & 3));
    const float bh = tc::to_tf32(vb), ah = tc::to_tf32(va);
    xh[off] = bh;
    xl[off] = tc::to_tf32(vb - bh);
    xh[aoff + off] = ah;
    xl[aoff + off] = tc::to_tf32(va - ah);
  }
  xn[i] = nrm;
}

__global__ void gram_tilemax_kernel(const float* __restrict__ xn, int n_pad, float* __restrict__ tmax) {
  const int jt = blockIdx.x * blockDim.x + threadIdx.x;
  if (jt * 64 >= n_pad) return;
  float m = 0.0f;
  for (int j = 0; j < 64; ++j) m = fmaxf(m, xn[jt * 64 + j]);
  tmax[jt] = m;
}

cudaError_t launch_gram_pack(const double* X, long long ldx, int n, int d, int n_pad, const double* ls,
                             double prescale, double* mu, float* xh, float* xl, float* xn, cudaStream_t st) {
  if (d < 1 || d > kGramMaxDim) return cudaErrorInvalidValue;
  gram_mean_kernel<<<d, 256, 0, st>>>(X, ldx, n, ls, mu);
  gram_pack_kernel<<<(n_pad + 127) / 128, 128, 0, st>>>(X, ldx, n, d, n_pad, ls, mu, sqrt(prescale), xh, xl, xn);
  const int nt = n_pad / 64;
  gram_tilemax_kernel<<<(nt + 127) / 128, 128, 0, st>>>(xn, n_pad, xn + n_pad);
  return cudaGetLastError();
}

int tcg_npad(int t) {
  static const int set[] = {1, 2, 4, 6, 7, 8, 9, 10, 12};
  const int need = (t + 7) / 8;
  for (int v : set)
    if (v >= need) return 8 * v;
  return -1;
}

// per column c < t: sigma_c = 2^(14 - e), max |V[:, c]| = m 2^e (m in [0.5, 1)), so
// |V sigma| < 2^14 and both fp16 halves stay in range; colscale_c = scale / (2^10 sigma_c).
// Column maxima: 2-D grid of row chunks, integer atomicMax on the (non-negative) fp64 bit
// patterns (order-independent, so deterministic); the pack kernel derives sigma from them.
__global__ void vmax_kernel(const double* __restrict__ V, long long ldv, int n, unsigned long long* __restrict__ vmax) {
  const int c = blockIdx.y;
  double m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    m = fmax(m, fabs(V[c * ldv + i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(vmax + c, static_cast<unsigned long long>(__double_as_longlong(m)));
}
GPK_DEV double sigma_of(unsigned long long bits) {
  const double m = __longlong_as_double(static_cast<long long>(bits));
  int e = 0;
  if (m > 0.0) frexp(m, &e);
  return ldexp(1.0, 14 - e);
}

// V (fp64, column-major) -> per 64-row j-tile, NPAD x 64 fp16 hi / lo tiles of V sigma
// in the 128B-swizzled K-major UMMA layout.
__global__ void pack_v_f16_kernel(const double* __restrict__ V, long long ldv, int t, int n, int n_pad, int npad,
                                  const unsigned long long* __restrict__ vmax, double scale,
                                  double* __restrict__ colscale, __half* __restrict__ vhi,
                                  __half* __restrict__ vlo) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long total = static_cast<long long>(n_pad) * npad;
  if (idx >= total) return;
  const int j = static_cast<int>(idx & 63);
  const long long rest = idx >> 6;
  const int c = static_cast<int>(rest % npad);
  const long long jt = rest / npad;
  const long long i = jt * 64 + j;
  const double sg = c < t ? sigma_of(vmax[c]) : 1.0;
  if (jt == 0 && j == 0 && c < t) colscale[c] = scale / (1024.0 * sg);
  const float v = (c < t && i < n) ? static_cast<float>(V[c * ldv + i] * sg) : 0.0f;
  const __half hi = __float2half_rn(v);
  const __half lo = __float2half_rn(v - __half2float(hi));
  const long long off = jt * npad * 64 + (c >> 3) * 512 + (c & 7) * 64 + (((j >> 3) ^ (c & 7)) << 3) + (j & 7);
  vhi[off] = hi;
  vlo[off] = lo;
}

cudaError_t launch_pack_v_f16(const double* V, long long ldv, int t, int n, int n_pad, int npad, double scale,
                              void* vmax, double* colscale, void* vhi, void* vlo, cudaStream_t st) {
  unsigned long long* vm = static_cast<unsigned long long*>(vmax);
  cudaError_t e = cudaMemsetAsync(vm, 0, sizeof(unsigned long long) * t, st);
  if (e != cudaSuccess) return e;
  const int bx = std::min(16, (n + 1023) / 1024);
  vmax_kernel<<<dim3(bx, t), 256, 0, st>>>(V, ldv, n, vm);
  const long long total = static_cast<long long>(n_pad) * npad;
  pack_v_f16_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      V, ldv, t, n, n_pad, npad, vm, scale, colscale, static_cast<__half*>(vhi), static_cast<__half*>(vlo));
  return cudaGetLastError();
}

// pack only, with column maxima already in vmax (the fused CG p-update computed them)
cudaError_t launch_pack_v_f16_only(const double* V, long long ldv, int t, int n, int n_pad, int npad, double scale,
                                   const void* vmax, double* colscale, void* vhi, void* vlo, cudaStream_t st) {
  const long long total = static_cast<long long>(n_pad) * npad;
  pack_v_f16_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      V, ldv, t, n, n_pad, npad, static_cast<const unsigned long long*>(vmax), scale, colscale,
      static_cast<__half*>(vhi), static_cast<__half*>(vlo));
  return cudaGetLastError();
}

cudaError_t launch_fused_kmvm_tcg(int family, int d, int direct_dp, const float* xh, const float* xl,
                                  const float* xn, const float* x32, const void* vhi, const void* vlo,
                                  const double* colscale, double* out, const MvmArgs& a, int splits,
                                  cudaStream_t st) {
  const int npad = tcg_npad(a.t);
  if (npad < 0 || d < 1 || d > 32 || (direct_dp == 0 && d > kGramMaxDim)) return cudaErrorInvalidValue;
  const int ks = (d + 2 + 7) / 8;  // Gram mode: the augmented coordinates [x~, 1, n] / [-2 x~, n, 1]
  const int units = (a.row_end - a.row_begin + tcg::BM - 1) / tcg::BM * splits;
  dim3 g(a.ctas > 0 ? std::min(units, a.ctas) : units);  // persistent grid, or one CTA per unit
  const int nc8 = npad / 8;
  const __half* h = static_cast<const __half*>(vhi);
  const __half* l = static_cast<const __half*>(vlo);
  const int dd = direct_dp;
  switch (family) {
    case kRBF: return tcg::launch_tcg_fam<kRBF>(ks, dd, nc8, xh, xl, xn, x32, h, l, colscale, out, a, g, st);
    case kMatern12: return tcg::launch_tcg_fam<kMatern12>(ks, dd, nc8, xh, xl, xn, x32, h, l, colscale, out, a, g, st);
    case kMatern32: return tcg::launch_tcg_fam<kMatern32>(ks, dd, nc8, xh, xl, xn, x32, h, l, colscale, out, a, g, st);
    case kMatern52: return tcg::launch_tcg_fam<kMatern52>(ks, dd, nc8, xh, xl, xn, x32, h, l, colscale, out, a, g, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace gpk

#ifdef GPK_TCG_TRACE
extern "C" int gpk_tcg_trace(long long* out, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, gpk::tcg::g_tcg_trace, sizeof(long long) * n));
}
#endif
