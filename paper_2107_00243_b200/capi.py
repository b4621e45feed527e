"""ctypes binding of libgpkrylov_cuda.so (include/gpkrylov_cuda.h).

The product path: every call goes to the sm_100a library.  There is no CPU
fallback — if the shared library is missing or no CUDA device is visible the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GPK_LIB_PATH") or os.path.join(_HERE, "lib", "libgpkrylov_cuda.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "gpkrylov_cuda.h")

GPK_OK, GPK_INPUT_ERROR, GPK_NUMERICAL_ERROR, GPK_SOLVER_ERROR, GPK_CUDA_ERROR, GPK_NCCL_ERROR = range(6)
GPK_RBF, GPK_MATERN12, GPK_MATERN32, GPK_MATERN52, GPK_RATQUAD = range(5)
GPK_PREC_FP64, GPK_PREC_FP32, GPK_PREC_TF32X3 = 0, 1, 2
GPK_MVM_AUTO, GPK_MVM_DIRECT, GPK_MVM_GRAM = 0, 1, 2


class gpk_cg_cfg(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("rel_tol", C.c_double), ("collect_tridiag", C.c_int),
                ("precision", C.c_int), ("refine", C.c_int)]


class gpk_mll_cfg(C.Structure):
    _fields_ = [("solver", gpk_cg_cfg), ("share_probes", C.c_int), ("with_gradient", C.c_int),
                ("backward_mode", C.c_int)]


class gpk_mll_result(C.Structure):
    _fields_ = [("value", C.c_double), ("gradient", C.POINTER(C.c_double)), ("solve_iterations", C.c_int),
                ("forward_gammas", C.POINTER(C.c_double)), ("backward_gammas", C.POINTER(C.c_double)),
                ("value_sample_variance", C.c_double), ("forward_cg_iterations", C.POINTER(C.c_int)),
                ("total_cg_iterations", C.c_int), ("logdet", C.c_double), ("logdet_precond", C.c_double),
                ("quad", C.c_double), ("refine_passes", C.c_int), ("max_true_rel_residual", C.c_double),
                ("seconds_solve", C.c_double), ("seconds_backward", C.c_double), ("seconds_total", C.c_double),
                ("kernel_entries", C.c_longlong), ("mvm_flops", C.c_longlong), ("gpu_launches", C.c_int),
                ("max_cg_rel_residual", C.c_double), ("unconverged_columns", C.c_int),
                ("backward_mode_used", C.c_int)]


class gpk_opt_options(C.Structure):
    _fields_ = [("method", C.c_int), ("max_steps", C.c_int), ("lbfgs_memory", C.c_int), ("armijo_c1", C.c_double),
                ("wolfe_c2", C.c_double), ("adam_lr", C.c_double), ("early_stop_patience", C.c_int),
                ("grad_tol", C.c_double), ("max_line_search", C.c_int)]


class gpk_opt_result(C.Structure):
    _fields_ = [("best_log_params", C.POINTER(C.c_double)), ("best_validation", C.c_double),
                ("final_train_neg_mll_per_point", C.c_double), ("final_objective", C.c_double),
                ("minimizer_steps", C.c_int), ("converged", C.c_int), ("stop_reason", C.c_int),
                ("n_steps", C.c_int), ("step_theta", C.POINTER(C.c_double)),
                ("step_objective", C.POINTER(C.c_double)), ("step_validation", C.POINTER(C.c_double)),
                ("step_wall_time", C.POINTER(C.c_double)), ("step_length", C.POINTER(C.c_double)),
                ("step_f_before", C.POINTER(C.c_double)), ("step_dir_derivative_before", C.POINTER(C.c_double)),
                ("step_dir_derivative_after", C.POINTER(C.c_double)), ("step_accepted", C.POINTER(C.c_int)),
                ("step_evaluations", C.POINTER(C.c_longlong)), ("eval_capacity", C.c_int),
                ("n_evaluations", C.c_int), ("eval_step", C.POINTER(C.c_int)), ("eval_f", C.POINTER(C.c_double)),
                ("eval_grad_norm", C.POINTER(C.c_double)), ("total_cg_iterations", C.c_longlong),
                ("seconds_total", C.c_double)]


GPK_OPT_LBFGS, GPK_OPT_ADAM = 0, 1
GPK_OPT_MAX_STEPS, GPK_OPT_GRAD_TOL, GPK_OPT_LINE_SEARCH_FAILED, GPK_OPT_STOPPED = range(4)

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_L = C.POINTER(C.c_int64)
_V = C.c_void_p

# name -> (restype, argtypes); mirrors include/gpkrylov_cuda.h
SIGNATURES = {
    "gpk_create": (C.c_int, [C.c_int, C.POINTER(_V)]),
    "gpk_destroy": (None, [_V]),
    "gpk_last_error": (C.c_char_p, [_V]),
    "gpk_version": (C.c_char_p, []),
    "gpk_set_data": (C.c_int, [_V, _D, C.c_int64, C.c_int64, C.c_int64]),
    "gpk_set_data_device": (C.c_int, [_V, _V, C.c_int64, C.c_int64, C.c_int64]),
    "gpk_set_params": (C.c_int, [_V, C.c_int, C.c_double, C.c_double, _D, C.c_double]),
    "gpk_kernel_mvm": (C.c_int, [_V, _D, C.c_int64, C.c_int, _D, C.c_int64, C.c_int]),
    "gpk_kernel_deriv_mvm": (C.c_int, [_V, C.c_int, _D, C.c_int64, C.c_int, _D, C.c_int64, C.c_int]),
    "gpk_kernel_column": (C.c_int, [_V, C.c_int64, _D]),
    "gpk_kernel_deriv_column": (C.c_int, [_V, C.c_int, C.c_int64, _D]),
    "gpk_precond_identity": (C.c_int, [_V]),
    "gpk_pivoted_cholesky": (C.c_int, [_V, C.c_int, C.c_double, C.c_double, _L, _I, _D]),
    "gpk_precond_deriv_factors": (C.c_int, [_V]),
    "gpk_precond_factor": (C.c_int, [_V, _D, C.c_int64]),
    "gpk_precond_deriv_factor": (C.c_int, [_V, C.c_int, _D, C.c_int64]),
    "gpk_precond_solve": (C.c_int, [_V, _D, C.c_int64, C.c_int, _D, C.c_int64]),
    "gpk_precond_logdet": (C.c_int, [_V, _D]),
    "gpk_precond_trace_inv_deriv": (C.c_int, [_V, C.c_int, _D]),
    "gpk_mbcg": (C.c_int, [_V, _D, C.c_int64, C.c_int, C.POINTER(gpk_cg_cfg), _D, C.c_int64, _I, _I, _D, _D, _D]),
    "gpk_evaluate_mll": (C.c_int, [_V, _D, _D, C.c_int64, C.c_int, C.c_uint64, C.POINTER(gpk_mll_cfg),
                                   C.POINTER(gpk_mll_result)]),
    "gpk_evaluate_mll_device": (C.c_int, [_V, _V, _V, C.c_int64, C.c_int, C.c_uint64, C.POINTER(gpk_mll_cfg),
                                          C.POINTER(gpk_mll_result)]),
    "gpk_make_probes": (C.c_int, [C.c_int64, C.c_int, C.c_uint64, _D]),
    "gpk_make_probes_device": (C.c_int, [_V, C.c_int64, C.c_int, C.c_uint64, C.c_void_p]),
    "gpk_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "gpk_set_mvm_variant": (C.c_int, [_V, C.c_int]),
    "gpk_get_mvm_variant": (C.c_int, [_V, _I, _D]),
    "gpk_launch_count": (C.c_longlong, [_V]),
    "gpk_stream": (_V, [_V]),
    "gpk_profile_enable": (C.c_int, [_V, C.c_int]),
    "gpk_profile_read": (C.c_int, [_V, C.c_int, _D, C.POINTER(C.c_longlong), _D, _D]),
    "gpk_profile_reset": (C.c_int, [_V]),
    "gpk_nccl_unique_id": (C.c_int, [_V]),
    "gpk_create_sharded": (C.c_int, [C.c_int, C.c_int, C.c_int, _V, C.POINTER(_V)]),
    "gpk_group_create": (C.c_int, [C.c_int, C.POINTER(_V)]),
    "gpk_group_destroy": (None, [_V]),
    "gpk_create_in_group": (C.c_int, [C.c_int, _V, C.c_int, C.POINTER(_V)]),
    "gpk_shard_rows": (C.c_int, [_V, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "gpk_data_shape": (C.c_int, [_V, C.POINTER(C.c_int64), _I]),
    "gpk_mll_exact": (C.c_int, [_V, _D, _D, _D]),
    "gpk_cross_kernel_mvm": (C.c_int, [_V, _D, C.c_int64, C.c_int64, _D, _D]),
    "gpk_predict_mean": (C.c_int, [_V, _D, _D, C.c_int64, C.c_int64, C.POINTER(gpk_cg_cfg), _D, _I]),
    "gpk_load_csv": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                               C.POINTER(_V), C.c_char_p, C.c_int64]),
    "gpk_dataset_free": (None, [_V]),
    "gpk_dataset_shape": (C.c_int, [_V, C.c_int, _L, _I]),
    "gpk_dataset_copy": (C.c_int, [_V, C.c_int, _D, C.c_int64, _D]),
    "gpk_dataset_stats": (C.c_int, [_V, _I, _D, _D, _D, _D]),
    "gpk_dataset_column_name": (C.c_char_p, [_V, C.c_int]),
    "gpk_dataset_invert": (C.c_int, [_V, _D, C.c_int64, C.c_int64, _D]),
    "gpk_optimize": (C.c_int, [_V, _D, _V, _D, C.c_int, C.c_int, _D, C.c_int, C.c_double, C.c_int,
                               C.POINTER(gpk_opt_options), C.POINTER(gpk_mll_cfg), C.c_uint64, C.c_int64,
                               C.POINTER(gpk_opt_result)]),
}


class ExtensionMissing(RuntimeError):
    pass


class _Stubbed:
    """An experiment build (GPK_LIB_PATH) missing some exports: the missing names raise
    ExtensionMissing naming the symbol at the call, every other attribute is the library's."""

    def __init__(self, handle, missing):
        self._h, self._missing = handle, set(missing)

    def __getattr__(self, name):
        if name in self._missing:
            def stub(*_a, **_k):
                raise ExtensionMissing(f"{LIB_PATH} does not export {name}")
            return stub
        return getattr(self._h, name)


_lib = None


def _preload_nccl():
    """The library links libnccl.so.2.  When PyTorch is installed its wheel bundles a (newer) NCCL
    under the same soname; whichever copy is loaded first serves both, and torch cannot import on
    top of an older system copy.  Load torch's copy first (if there is one) so that the import
    order of torch and this package does not matter."""
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
        for base in (spec.submodule_search_locations if spec else []):
            so = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(so):
                C.CDLL(so, mode=C.RTLD_GLOBAL)
                return
    except Exception:
        pass  # the system libnccl.so.2 on the loader path is used


def lib():
    """Load the sm_100a library (raises if it was not built; never falls back)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        _preload_nccl()
        handle = C.CDLL(LIB_PATH)
        missing = []
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name, None)
            if fn is None:
                if not os.environ.get("GPK_LIB_PATH"):
                    raise ExtensionMissing(f"{LIB_PATH} does not export {name}")
                missing.append(name)  # an older experiment build: bound to a stub that raises
                continue
            fn.restype = res
            fn.argtypes = args
        if missing:
            import warnings

            warnings.warn(f"GPK_LIB_PATH={LIB_PATH} lacks {len(missing)} exports: {', '.join(missing)}")
            handle = _Stubbed(handle, missing)
        _lib = handle
    return _lib


def header_functions():
    """Function names declared in include/gpkrylov_cuda.h."""
    src = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:gpk_status|void\*?|const char\*|uint64_t|long long)\s+(gpk_\w+)\s*\(",
                                 src, flags=re.M)))
