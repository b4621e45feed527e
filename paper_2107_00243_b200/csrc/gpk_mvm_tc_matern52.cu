// tcgen05 fused kernel-MVM instantiations for one kernel family (see gpk_mvm_tc.cuh).
#include "gpk_mvm_tc.cuh"
GPK_INSTANTIATE_TC_FAMILY(gpk::kMatern52)
