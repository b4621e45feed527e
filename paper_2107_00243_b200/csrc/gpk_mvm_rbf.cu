// Fused kernel-MVM instantiations for one kernel family (see gpk_mvm.cuh).
#include "gpk_mvm_dispatch.cuh"
GPK_INSTANTIATE_FAMILY(gpk::kRBF)
