// Front end of the tcgen05 fused MVM: V packing (tf32 hi/lo, 128B-swizzled
// K-major tiles) and dispatch.
#include "gpk_mvm_tc.cuh"

namespace gpk {
namespace tc {
template <int FAM>
cudaError_t launch_tc_fam(int dp, int nc8, const float* X, const float* Vhi, const float* Vlo, double* out,
                          const MvmArgs& a, dim3 g, cudaStream_t st);
}

int tc_npad(int t) {
  static const int set[] = {1, 2, 4, 6, 7, 8, 9, 10, 12, 16};
  const int need = (t + 7) / 8;
  for (int s : set)
    if (s >= need) return 8 * s;
  return -1;
}

// V (fp64, column-major, t columns) -> per 32-row j-tile, NPAD x 32 tf32 hi / lo
// tiles in the canonical 128B-swizzled K-major UMMA layout (so one bulk copy
// yields the smem image the tensor core expects).
__global__ void pack_v_tc_kernel(const double* __restrict__ V, long long ldv, int t, int n, int n_pad, int npad,
                                 float* __restrict__ vhi, float* __restrict__ vlo) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long total = static_cast<long long>(n_pad) * npad;
  if (idx >= total) return;
  const int j = static_cast<int>(idx & 31);
  const long long rest = idx >> 5;
  const int c = static_cast<int>(rest % npad);
  const int jt = static_cast<int>(rest / npad);
  const int i = jt * 32 + j;
  const float v = (c < t && i < n) ? static_cast<float>(V[c * ldv + i]) : 0.0f;
  const float hi = tc::to_tf32(v);
  const float lo = tc::to_tf32(v - hi);
  const long long off = static_cast<long long>(jt) * npad * 32 + (c >> 3) * 256 + (c & 7) * 32 +
                        ((((j >> 2) ^ (c & 7))) << 2) + (j & 3);
  vhi[off] = hi;
  vlo[off] = lo;
}

cudaError_t launch_pack_v_tc(const double* V, long long ldv, int t, int n, int n_pad, int npad, float* vhi,
                             float* vlo, cudaStream_t st) {
  const long long total = static_cast<long long>(n_pad) * npad;
  pack_v_tc_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(V, ldv, t, n, n_pad, npad, vhi, vlo);
  return cudaGetLastError();
}

cudaError_t launch_fused_kmvm_tc(int family, int dp, const float* X, const float* vhi, const float* vlo, double* out,
                                 const MvmArgs& a, int splits, cudaStream_t st) {
  const int npad = tc_npad(a.t);
  if (npad < 0) return cudaErrorInvalidValue;
  dim3 g((a.row_end - a.row_begin + tc::BM - 1) / tc::BM, splits);
  const int nc8 = npad / 8;
  switch (family) {
    case kRBF: return tc::launch_tc_fam<kRBF>(dp, nc8, X, vhi, vlo, out, a, g, st);
    case kMatern12: return tc::launch_tc_fam<kMatern12>(dp, nc8, X, vhi, vlo, out, a, g, st);
    case kMatern32: return tc::launch_tc_fam<kMatern32>(dp, nc8, X, vhi, vlo, out, a, g, st);
    case kMatern52: return tc::launch_tc_fam<kMatern52>(dp, nc8, X, vhi, vlo, out, a, g, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace gpk
