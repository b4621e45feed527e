// Template dispatch for the fused kernel MVM; included once per kernel family
// (gpk_mvm_<family>.cu) so the instantiations compile in parallel.
#pragma once
#include "gpk_mvm.cuh"

namespace gpk {

template <int FAM, typename T, int DP, int MODE>
cudaError_t dispatch_tn(int tn, const void* X, const void* V, double* out, const MvmArgs& a, dim3 g,
                        cudaStream_t st) {
  const T* x = static_cast<const T*>(X);
  const T* v = static_cast<const T*>(V);
#define GPK_TN(N) \
  case N: return launch_fused_kmvm_t<T, FAM, DP, N, MODE>(x, v, out, a, g, st);
  if constexpr (sizeof(T) == 4 && MODE == kModeValue) {
    switch (tn) {
      GPK_TN(1) GPK_TN(2) GPK_TN(3) GPK_TN(4) GPK_TN(5) GPK_TN(6) GPK_TN(7) GPK_TN(8) GPK_TN(9) GPK_TN(10)
      GPK_TN(12) GPK_TN(16)
      default: break;
    }
  } else if constexpr (sizeof(T) == 4) {
    switch (tn) {
      GPK_TN(1) GPK_TN(2) GPK_TN(4) GPK_TN(8) GPK_TN(16)
      default: break;
    }
  } else {
    switch (tn) {
      GPK_TN(1) GPK_TN(2) GPK_TN(4) GPK_TN(8)
      default: break;
    }
  }
#undef GPK_TN
  return cudaErrorInvalidValue;
}

template <int FAM, typename T, int MODE>
cudaError_t dispatch_dp(int dp, int tn, const void* X, const void* V, double* out, const MvmArgs& a, dim3 g,
                        cudaStream_t st) {
  switch (dp) {
    case 4: return dispatch_tn<FAM, T, 4, MODE>(tn, X, V, out, a, g, st);
    case 12: return dispatch_tn<FAM, T, 12, MODE>(tn, X, V, out, a, g, st);
    case 20: return dispatch_tn<FAM, T, 20, MODE>(tn, X, V, out, a, g, st);
    case 32: return dispatch_tn<FAM, T, 32, MODE>(tn, X, V, out, a, g, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int FAM>
cudaError_t launch_fused_kmvm_fam(bool fp64, int dp, int mode, int tn, const void* X, const void* V, double* out,
                                  const MvmArgs& a, dim3 g, cudaStream_t st) {
  if (fp64) {
    return mode == kModeValue ? dispatch_dp<FAM, double, kModeValue>(dp, tn, X, V, out, a, g, st)
                              : dispatch_dp<FAM, double, kModeDls>(dp, tn, X, V, out, a, g, st);
  }
  return mode == kModeValue ? dispatch_dp<FAM, float, kModeValue>(dp, tn, X, V, out, a, g, st)
                            : dispatch_dp<FAM, float, kModeDls>(dp, tn, X, V, out, a, g, st);
}

}  // namespace gpk

#define GPK_INSTANTIATE_FAMILY(FAM)                                                                        \
  namespace gpk {                                                                                          \
  template cudaError_t launch_fused_kmvm_fam<FAM>(bool, int, int, int, const void*, const void*, double*, \
                                                  const MvmArgs&, dim3, cudaStream_t);                    \
  }
