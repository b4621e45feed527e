// Tensor-core MVM instantiations for Matern-1/2 (direct-difference mode only, see gpk_mvm_tcg.cuh).
#include "gpk_mvm_tcg.cuh"
GPK_INSTANTIATE_TCG_FAMILY(gpk::kMatern12)
