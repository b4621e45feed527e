// Front end of the Gram-variant tensor-core MVM (gpk_mvm_tcg.cuh): packing of
// the centred, pre-scaled coordinates into tf32 hi/lo 128B-swizzled K-major
// tiles plus their fp32 squared norms, and dispatch.
#include "gpk_mvm_tcg.cuh"

namespace gpk {
namespace tcg {
template <int FAM>
cudaError_t launch_tcg_fam(int ks, int nc8, const float* Xh, const float* Xl, const float* Xn, const float* X32,
                           const float* Vhi,
                           const float* Vlo, double* out, const MvmArgs& a, dim3 g, cudaStream_t st);
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

// one thread per (row, coordinate slot): x~ = (X/l - mu) sqrt(prescale), split into
// tf32 hi / lo at the swizzled position of the tile image; padded rows and
// coordinates are zero.  Norms: fp32 sum of squares of the fp32 coordinates.
__global__ void gram_pack_kernel(const double* __restrict__ X, long long ldx, int n, int d, int n_pad,
                                 const double* __restrict__ ls, const double* __restrict__ mu, double pre,
                                 float* __restrict__ xh, float* __restrict__ xl, float* __restrict__ xn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  const long long tile = i >> 5;
  const int r = i & 31;
  float nrm = 0.0f;
  for (int k = 0; k < 32; ++k) {
    float v = 0.0f;
    if (i < n && k < d) v = static_cast<float>((X[k * ldx + i] / ls[k] - mu[k]) * pre);
    const float hi = tc::to_tf32(v);
    const float lo = tc::to_tf32(v - hi);
    const long long off = tile * 1024 + ((r >> 3) * 256 + (r & 7) * 32 + ((((k >> 2) ^ (r & 7))) << 2) + (k & 3));
    xh[off] = hi;
    xl[off] = lo;
    nrm = fmaf(v, v, nrm);
  }
  xn[i] = nrm;
}

cudaError_t launch_gram_pack(const double* X, long long ldx, int n, int d, int n_pad, const double* ls,
                             double prescale, double* mu, float* xh, float* xl, float* xn, cudaStream_t st) {
  if (d < 1 || d > 32) return cudaErrorInvalidValue;
  gram_mean_kernel<<<d, 256, 0, st>>>(X, ldx, n, ls, mu);
  gram_pack_kernel<<<(n_pad + 127) / 128, 128, 0, st>>>(X, ldx, n, d, n_pad, ls, mu, sqrt(prescale), xh, xl, xn);
  return cudaGetLastError();
}

cudaError_t launch_fused_kmvm_tcg(int family, int d, const float* xh, const float* xl, const float* xn,
                                  const float* x32, const float* vhi, const float* vlo, double* out, const MvmArgs& a, int splits,
                                  cudaStream_t st) {
  const int npad = tc_npad(a.t);
  if (npad < 0 || d < 1 || d > 32) return cudaErrorInvalidValue;
  const int ks = (d + 7) / 8;
  dim3 g((a.row_end - a.row_begin + tc::BM - 1) / tc::BM, splits);
  const int nc8 = npad / 8;
  switch (family) {
    case kRBF: return tcg::launch_tcg_fam<kRBF>(ks, nc8, xh, xl, xn, x32, vhi, vlo, out, a, g, st);
    case kMatern32: return tcg::launch_tcg_fam<kMatern32>(ks, nc8, xh, xl, xn, x32, vhi, vlo, out, a, g, st);
    case kMatern52: return tcg::launch_tcg_fam<kMatern52>(ks, nc8, xh, xl, xn, x32, vhi, vlo, out, a, g, st);
  }
  return cudaErrorInvalidValue;  // Matern-1/2 stays on the direct-difference kernels
}

}  // namespace gpk

#ifdef GPK_TCG_TRACE
extern "C" int gpk_tcg_trace(long long* out, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, gpk::tcg::g_tcg_trace, sizeof(long long) * n));
}
#endif
