// Gram-variant tensor-core MVM instantiations for one kernel family (see gpk_mvm_tcg.cuh).
#include "gpk_mvm_tcg.cuh"
GPK_INSTANTIATE_TCG_FAMILY(gpk::kRBF)
