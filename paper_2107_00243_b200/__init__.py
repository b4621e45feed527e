"""B200-native (sm_100a) preconditioned mBCG hot path of Wenger et al. (arXiv 2107.00243).

One log-marginal-likelihood + gradient evaluation (reference: evaluate_mll,
proj/include/gpkrylov/gp_likelihood.hpp:51-103) runs as hand-written CUDA
kernels behind the C-ABI in include/gpkrylov_cuda.h (libgpkrylov_cuda.so);
``gpkrylov`` mirrors the reference's C++ interface on top of it.
"""
from .gpkrylov import (  # noqa: F401
    CgConfig, CgResult, CudaError, DiagPlusLowRank, Hyperparameters, IdentityPreconditioner, InputError,
    KernelOperator, KernelSpec, MllConfig, MllEvaluation, NumericalError, ProbeBatch, SolverError, SymTridiagonal,
    batched_pcg, evaluate_mll, evaluate_mll_device, make_probes, make_probes_device, mix_seed, mll_estimate, mll_gradient, pcg_solve,
    pivoted_cholesky, pivoted_cholesky_deriv_factors, pivoted_cholesky_with_derivatives,
)
from .gpkrylov import (  # noqa: F401  SURVEY §8(f): the callers of the hot path
    DataSplits, Dataset, ExactMll, SplitFractions, Standardizer, load_csv, IdentityBuilder, OptimizeResult, OptOptions, PivotedCholeskyBuilder, count_model_evaluations,
    cross_kernel_mvm, mll_exact, optimize, predict_mean, run_training_arm,
)

__version__ = "0.1.0"
