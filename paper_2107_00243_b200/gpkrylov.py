"""Python mirror of the reference's gpkrylov interface over the sm_100a C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/gpkrylov (cited per symbol) so that callers and
tests read like the reference's own.  Matrices are numpy float64; the device
side lives in one ``gpk_ctx`` per KernelOperator.  Exceptions mirror
common.hpp:19-35: InputError (input_error), NumericalError (numerical_error),
SolverError (solver_error, a NumericalError).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import capi

# ---------------------------------------------------------------------------
# errors (common.hpp:19-35)
# ---------------------------------------------------------------------------


class GpkError(RuntimeError):
    status = -1


class InputError(GpkError, ValueError):
    status = capi.GPK_INPUT_ERROR


class NumericalError(GpkError):
    status = capi.GPK_NUMERICAL_ERROR


class SolverError(NumericalError):
    status = capi.GPK_SOLVER_ERROR


class CudaError(NumericalError):
    status = capi.GPK_CUDA_ERROR


_ERRS = {capi.GPK_INPUT_ERROR: InputError, capi.GPK_NUMERICAL_ERROR: NumericalError,
         capi.GPK_SOLVER_ERROR: SolverError, capi.GPK_CUDA_ERROR: CudaError, capi.GPK_NCCL_ERROR: NumericalError}


def _check(rc: int, ctx=None, what=""):
    if rc != capi.GPK_OK:
        msg = capi.lib().gpk_last_error(ctx).decode() if ctx is not None else what
        raise _ERRS.get(rc, GpkError)(msg or what)


_Dp = C.POINTER(C.c_double)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_Dp)


def _fcol(a) -> np.ndarray:
    """Column-major float64 (Eigen layout); 1-d inputs become one column."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a[:, None]
    return np.asfortranarray(a)


# ---------------------------------------------------------------------------
# kernels.hpp
# ---------------------------------------------------------------------------
FAMILIES = {"rbf": capi.GPK_RBF, "matern12": capi.GPK_MATERN12, "matern32": capi.GPK_MATERN32,
            "matern52": capi.GPK_MATERN52, "ratquad": capi.GPK_RATQUAD}


@dataclass
class KernelSpec:
    """kernels.hpp:70-87"""
    family: str = "rbf"
    ard: bool = True
    ratquad_alpha: float = 1.0

    @property
    def code(self) -> int:
        if isinstance(self.family, int):
            return self.family
        return FAMILIES[self.family]


@dataclass
class Hyperparameters:
    """Log-space hyperparameters, flat order (outputscale, lengthscale_0..d-1, noise) (kernels.hpp:17-64)."""
    log_outputscale: float = 0.0
    log_lengthscales: np.ndarray = field(default_factory=lambda: np.zeros(1))
    log_noise: float = math.log(1e-2)

    @staticmethod
    def from_raw(d, outputscale=1.0, lengthscale=1.0, noise=1e-2, lengthscales=None):
        ls = np.full(d, lengthscale, float) if lengthscales is None else np.asarray(lengthscales, float)
        return Hyperparameters(math.log(outputscale), np.log(ls), math.log(noise))

    def dim(self):
        return len(self.log_lengthscales)

    def num_params(self):
        return self.dim() + 2

    def outputscale(self):
        return math.exp(self.log_outputscale)

    def lengthscales(self):
        return np.exp(self.log_lengthscales)

    def noise_variance(self):
        return math.exp(self.log_noise)

    def raw_value(self, which):  # kernels.hpp:31-36
        if which == 0:
            return self.outputscale()
        if 1 <= which <= self.dim():
            return math.exp(self.log_lengthscales[which - 1])
        if which == self.dim() + 1:
            return self.noise_variance()
        raise InputError("Hyperparameters: parameter index out of range")

    def to_log_vector(self):
        return np.concatenate([[self.log_outputscale], self.log_lengthscales, [self.log_noise]])

    @staticmethod
    def from_log_vector(v):
        v = np.asarray(v, float)
        if v.size < 3:
            raise InputError("Hyperparameters: log vector needs at least 3 entries")
        return Hyperparameters(float(v[0]), v[1:-1].copy(), float(v[-1]))


def kOutputscaleIndex():
    return 0


def lengthscale_index(j):
    return 1 + j


def noise_index(d):
    return d + 1


class RankGroup:
    """In-process group of `world` ranks (one host thread per rank) for the row-sharded path;
    collectives are host-staged, so it runs on any number of devices (also one)."""

    def __init__(self, world: int):
        self.lib = capi.lib()
        g = C.c_void_p()
        _check(self.lib.gpk_group_create(int(world), C.byref(g)), None, "gpk_group_create failed")
        self.g = g
        self.world = int(world)

    def __del__(self):
        try:
            if getattr(self, "g", None):
                self.lib.gpk_group_destroy(self.g)
                self.g = None
        except Exception:
            pass


class _Ctx:
    """Owns one gpk_ctx (device state: data, packed operands, preconditioner, workspaces).
    shard=(RankGroup, rank) or ("nccl", rank, world, unique_id_bytes) makes it one rank of a
    row-sharded evaluation."""

    def __init__(self, device=0, shard=None):
        self.lib = capi.lib()
        h = C.c_void_p()
        if shard is None:
            rc = self.lib.gpk_create(int(device), C.byref(h))
        elif isinstance(shard[0], RankGroup):
            self.group = shard[0]  # keep the group alive
            rc = self.lib.gpk_create_in_group(int(device), shard[0].g, int(shard[1]), C.byref(h))
        else:
            _, rank, world, uid = shard
            buf = C.create_string_buffer(bytes(uid), 128)
            rc = self.lib.gpk_create_sharded(int(device), int(rank), int(world), buf, C.byref(h))
        if rc != capi.GPK_OK:
            raise CudaError(f"gpk_create(device={device}) failed with status {rc}: no usable CUDA device")
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.gpk_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def check(self, rc):
        _check(rc, self.h)


PREC = {"fp64": capi.GPK_PREC_FP64, "fp32": capi.GPK_PREC_FP32, "tf32x3": capi.GPK_PREC_TF32X3}


class KernelOperator:
    """Matrix-free K_hat = K + sigma^2 I on the GPU (kernels.hpp:157-336).

    Holds X on the device.  ``with_params`` moves the operator to new
    hyperparameters while keeping the attached preconditioner (the line-search
    situation of optimizer.hpp:437 vs :450-451)."""

    def __init__(self, spec: KernelSpec, x, params: Hyperparameters, device: int = 0, precision="fp64", shard=None):
        x = np.asfortranarray(np.asarray(x, dtype=np.float64))
        if x.ndim != 2 or x.shape[0] < 1:
            raise InputError("KernelOperator: empty dataset")
        if params.dim() != x.shape[1]:
            raise InputError("KernelOperator: lengthscale count must equal data dimension")
        self.spec = spec
        self._x = x
        self.params = params
        self.precision = precision
        self.ctx = _Ctx(device, shard)
        self.ctx.check(self.ctx.lib.gpk_set_data(self.ctx.h, _ptr(x), x.shape[0], x.shape[1], x.shape[0]))
        self._set_params(params)
        self.preconditioner = None

    def _set_params(self, params: Hyperparameters):
        ls = np.ascontiguousarray(params.log_lengthscales, dtype=np.float64)
        if ls.size != self._x.shape[1]:
            raise InputError("KernelOperator: lengthscale count must equal data dimension")
        self.ctx.check(self.ctx.lib.gpk_set_params(self.ctx.h, self.spec.code, float(self.spec.ratquad_alpha),
                                                   float(params.log_outputscale), _ptr(ls), float(params.log_noise)))
        self.params = params

    def with_params(self, params: Hyperparameters):
        self._set_params(params)
        return self

    MVM_VARIANTS = {"auto": 0, "direct": 1, "gram": 2}

    def set_mvm_variant(self, variant: str):
        """Kernel-entry strategy of the tensor-core MVM (gpk_set_mvm_variant): "auto", "direct", "gram"."""
        self.ctx.check(self.ctx.lib.gpk_set_mvm_variant(self.ctx.h, self.MVM_VARIANTS[variant]))
        return self

    def mvm_variant(self):
        """(variant in use: "direct" | "gram", max squared norm of the centred pre-scaled coordinates)."""
        v, m = C.c_int(), C.c_double()
        self.ctx.check(self.ctx.lib.gpk_get_mvm_variant(self.ctx.h, C.byref(v), C.byref(m)))
        return ("direct", "direct", "gram")[v.value], m.value

    def rows(self):
        return self._x.shape[0]

    def dim(self):
        return self._x.shape[1]

    def num_params(self):
        return self.dim() + 2

    def data(self):
        return self._x

    def _mvm(self, which, v, precision):
        vv = _fcol(v)
        if vv.shape[0] != self.rows():
            raise InputError("KernelOperator: vector length does not match n")
        out = np.empty_like(vv, order="F")
        p = PREC[precision or self.precision]
        if which < 0:
            rc = self.ctx.lib.gpk_kernel_mvm(self.ctx.h, _ptr(vv), vv.shape[0], vv.shape[1], _ptr(out), out.shape[0], p)
        else:
            rc = self.ctx.lib.gpk_kernel_deriv_mvm(self.ctx.h, int(which), _ptr(vv), vv.shape[0], vv.shape[1],
                                                   _ptr(out), out.shape[0], p)
        self.ctx.check(rc)
        return out[:, 0] if np.ndim(v) == 1 else out

    def apply(self, v, precision=None):
        """(K + sigma^2 I) v (kernels.hpp:184-195)"""
        return self._mvm(-1, v, precision)

    apply_matrix = apply

    def deriv_apply(self, which, v, precision=None):
        """(d K_hat / d theta_which) v, raw parameter (kernels.hpp:205-215)"""
        if which < 0 or which > self.dim() + 1:
            raise InputError("KernelOperator: hyperparameter index out of range")
        return self._mvm(which, v, precision)

    deriv_apply_matrix = deriv_apply

    def shard_rows(self):
        """This rank's [r0, r1) rows of the n-length arrays (the whole range when unsharded)."""
        a, b = C.c_int64(), C.c_int64()
        self.ctx.check(self.ctx.lib.gpk_shard_rows(self.ctx.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def kernel_diagonal(self):  # kernels.hpp:230-233
        return np.full(self.rows(), self.params.outputscale() ** 2)

    def kernel_column(self, i):  # kernels.hpp:235-243
        out = np.empty(self.rows())
        self.ctx.check(self.ctx.lib.gpk_kernel_column(self.ctx.h, int(i), _ptr(out)))
        return out

    def kernel_deriv_diagonal(self, which):  # kernels.hpp:245-250
        if which < 0 or which > self.dim() + 1:
            raise InputError("KernelOperator: hyperparameter index out of range")
        return np.full(self.rows(), 2.0 * self.params.outputscale() if which == 0 else 0.0)

    def kernel_deriv_column(self, which, i):  # kernels.hpp:252-267
        out = np.empty(self.rows())
        self.ctx.check(self.ctx.lib.gpk_kernel_deriv_column(self.ctx.h, int(which), int(i), _ptr(out)))
        return out


# ---------------------------------------------------------------------------
# preconditioners.hpp / common.hpp
# ---------------------------------------------------------------------------
class IdentityPreconditioner:
    """common.hpp:59-70 — installs P = I on the operator's device context."""

    def __init__(self, op: KernelOperator):
        self.op = op
        op.ctx.check(op.ctx.lib.gpk_precond_identity(op.ctx.h))
        op.preconditioner = self

    def logdet(self):
        return 0.0

    def solve(self, v):
        return np.array(v, dtype=np.float64, copy=True)

    def trace_inv_deriv(self, which):
        return 0.0

    def has_derivatives(self):
        return True


class DiagPlusLowRank:
    """P_hat = sigma^2 I + L L^T with Woodbury solves, resident on the operator's device
    (preconditioners.hpp:82-186).  Built by ``pivoted_cholesky``."""

    def __init__(self, op: KernelOperator, noise, rank, pivots):
        self.op = op
        self._noise = noise
        self._rank = rank
        self._pivots = pivots
        self._has_deriv = False

    def rows(self):
        return self.op.rows()

    def rank(self):
        return self._rank

    def noise_variance(self):
        return self._noise

    def pivots(self):
        return list(self._pivots)

    def _ctx(self):
        if self.op.preconditioner is not self:
            raise InputError("DiagPlusLowRank: preconditioner was replaced on this operator")
        return self.op.ctx

    def factor(self):
        c = self._ctx()
        out = np.zeros((self.rows(), self._rank), order="F")
        c.check(c.lib.gpk_precond_factor(c.h, _ptr(out), self.rows()))
        return out

    def solve(self, v):
        """P^{-1} v (:114-118)"""
        c = self._ctx()
        vv = _fcol(v)
        out = np.empty_like(vv, order="F")
        c.check(c.lib.gpk_precond_solve(c.h, _ptr(vv), vv.shape[0], vv.shape[1], _ptr(out), out.shape[0]))
        return out[:, 0] if np.ndim(v) == 1 else out

    solve_matrix = solve

    def logdet(self):
        c = self._ctx()
        out = C.c_double()
        c.check(c.lib.gpk_precond_logdet(c.h, C.byref(out)))
        return out.value

    def has_derivatives(self):
        return self._has_deriv

    def deriv_factor(self, which):
        c = self._ctx()
        out = np.zeros((self.rows(), self._rank), order="F")
        c.check(c.lib.gpk_precond_deriv_factor(c.h, int(which), _ptr(out), self.rows()))
        return out

    def trace_inv_deriv(self, which):
        """tr(P^{-1} dP/dtheta_which) (:138-145, :168)"""
        c = self._ctx()
        out = C.c_double()
        c.check(c.lib.gpk_precond_trace_inv_deriv(c.h, int(which), C.byref(out)))
        return out.value


def pivoted_cholesky(op: KernelOperator, rank: int, diag_tol: float = 0.0, noise_variance: Optional[float] = None,
                     want_remaining: bool = False):
    """Greedy pivoted partial Cholesky of the noise-free K in fp64 (preconditioners.hpp:236-264)."""
    noise = op.params.noise_variance() if noise_variance is None else float(noise_variance)
    piv = np.zeros(max(int(rank), 1), dtype=np.int64)
    ach = C.c_int()
    rem = np.zeros(op.rows()) if want_remaining else None
    op.ctx.check(op.ctx.lib.gpk_pivoted_cholesky(op.ctx.h, int(rank), float(diag_tol), noise,
                                                 piv.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(ach), _ptr(rem)))
    p = DiagPlusLowRank(op, noise, ach.value, piv[: ach.value].tolist())
    op.preconditioner = p
    return (p, rem) if want_remaining else p


def pivoted_cholesky_deriv_factors(op: KernelOperator, p: DiagPlusLowRank):
    """Frozen-pivot dL/dtheta (preconditioners.hpp:269-295), kept on the device."""
    c = p._ctx()
    c.check(c.lib.gpk_precond_deriv_factors(c.h))
    p._has_deriv = True
    return p


def pivoted_cholesky_with_derivatives(op: KernelOperator, rank: int, diag_tol: float = 0.0):
    """preconditioners.hpp:299-305 / build_preconditioner's pivoted-Cholesky branch (experiments.hpp:37-38, :59-61)."""
    p = pivoted_cholesky(op, rank, diag_tol, op.params.noise_variance())
    return pivoted_cholesky_deriv_factors(op, p)


# ---------------------------------------------------------------------------
# krylov.hpp
# ---------------------------------------------------------------------------
@dataclass
class CgConfig:
    """krylov.hpp:15-24 (+ GPU fields: operator precision, fp64 defect-correction passes)."""
    max_iters: int = 100
    rel_tol: float = 1e-6
    collect_tridiag: bool = False
    precision: str = "tf32x3"
    refine: int = 2

    def c(self):
        return capi.gpk_cg_cfg(int(self.max_iters), float(self.rel_tol), int(self.collect_tridiag),
                               PREC[self.precision], int(self.refine))


@dataclass
class SymTridiagonal:
    diag: np.ndarray
    subdiag: np.ndarray

    def size(self):
        return len(self.diag)


@dataclass
class CgResult:
    """krylov.hpp:33-39"""
    solution: np.ndarray
    iterations_used: int = 0
    converged: bool = False
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    tridiag: Optional[SymTridiagonal] = None


def batched_pcg(op: KernelOperator, B, prec, cfg: CgConfig) -> list:
    """Independent PCG solves for the columns of B in ONE batched device solve (krylov.hpp:133-153)."""
    if prec is None or op.preconditioner is not prec:
        raise InputError("batched_pcg: preconditioner is not attached to this operator")
    Bm = _fcol(B)
    if Bm.shape[0] != op.rows():
        raise InputError("batched_pcg: rhs rows do not match operator")
    t = Bm.shape[1]
    X = np.zeros_like(Bm, order="F")
    mi = int(cfg.max_iters)
    it = np.zeros(t, dtype=np.int32)
    cv = np.zeros(t, dtype=np.int32)
    ah = np.zeros((mi, t), order="F")
    bh = np.zeros((mi, t), order="F")
    rh = np.zeros((mi, t), order="F")
    cc = cfg.c()
    op.ctx.check(op.ctx.lib.gpk_mbcg(op.ctx.h, _ptr(Bm), Bm.shape[0], t, C.byref(cc), _ptr(X), X.shape[0],
                                     it.ctypes.data_as(C.POINTER(C.c_int)), cv.ctypes.data_as(C.POINTER(C.c_int)),
                                     _ptr(ah), _ptr(bh), _ptr(rh)))
    out = []
    for c in range(t):
        m = int(it[c])
        tri = None
        if cfg.collect_tridiag:  # krylov.hpp:85-92
            a, b = ah[:m, c], bh[: max(m - 1, 0), c]
            dg = 1.0 / a
            if m > 1:
                dg[1:] += b / a[:-1]
            tri = SymTridiagonal(dg, np.sqrt(b) / a[:-1] if m > 1 else np.zeros(0))
        out.append(CgResult(X[:, c].copy(), m, bool(cv[c]), rh[:m, c].copy(), tri))
    return out


def pcg_solve(op: KernelOperator, b, prec, cfg: CgConfig) -> CgResult:
    """krylov.hpp:47-129"""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 1 or b.shape[0] != op.rows():
        raise InputError("pcg_solve: rhs length does not match operator")
    try:
        return batched_pcg(op, b[:, None], prec, cfg)[0]
    except SolverError as e:
        msg = str(e)
        prefix = "batched_pcg: column 0: "
        raise SolverError(msg[len(prefix):] if msg.startswith(prefix) else msg) from None


# ---------------------------------------------------------------------------
# trace_estimation.hpp
# ---------------------------------------------------------------------------
@dataclass
class ProbeBatch:
    probes: np.ndarray
    seed: int = 0
    count: int = 0


def mix_seed(seed: int, salt: int) -> int:
    """common.hpp:93-98"""
    return int(capi.lib().gpk_mix_seed(C.c_uint64(seed), C.c_uint64(salt)))


def make_probes(n: int, count: int, seed: int) -> ProbeBatch:
    """trace_estimation.hpp:27-36 — normalised Rademacher probes from std::mt19937_64(seed)."""
    if n < 1:
        raise InputError("make_probes: n must be >= 1")
    if count < 1:
        raise InputError("make_probes: need at least one probe")
    z = np.empty((n, count), order="F")
    _check(capi.lib().gpk_make_probes(int(n), int(count), C.c_uint64(seed), _ptr(z)), None, "make_probes failed")
    return ProbeBatch(z, int(seed), int(count))


def make_probes_device(k: "KernelOperator", count: int, seed: int, device=0):
    """The same stream generated by the device kernel (gpk_probes.cu) on the operator's stream,
    into a torch cuda tensor of shape (count, n) -- column c of the reference's n x count block is
    row c (the layout evaluate_mll_device takes); bitwise make_probes."""
    import torch

    n = k.rows()
    if count < 1:
        raise InputError("make_probes: need at least one probe")
    z = torch.empty((count, n), dtype=torch.float64, device=f"cuda:{device}")
    k.ctx.check(k.ctx.lib.gpk_make_probes_device(k.ctx.h, int(n), int(count), C.c_uint64(seed),
                                                 C.c_void_p(z.data_ptr())))

    torch.cuda.synchronize()  # the library stream is not torch's: the caller may read z right away
    return z


# ---------------------------------------------------------------------------
# gp_likelihood.hpp
# ---------------------------------------------------------------------------
@dataclass
class MllConfig:
    """gp_likelihood.hpp:26-32 (+ backward: 'fused' bilinear derivative pass, 'faithful' per-RHS
    solves, 'auto' = fused when every forward solve converged, else faithful, or
    'fused_per_probe' = fused + per-probe backward gammas from (d+1) derivative MVMs)."""
    solver: CgConfig = field(default_factory=CgConfig)
    share_probes: bool = True
    backward: str = "auto"

    def c(self, with_gradient):
        modes = {"fused": 0, "faithful": 1, "auto": 2, "fused_per_probe": 3}
        if self.backward not in modes:
            raise InputError(f"MllConfig: unknown backward mode {self.backward!r}")
        return capi.gpk_mll_cfg(self.solver.c(), int(self.share_probes), int(with_gradient), modes[self.backward])


@dataclass
class MllEvaluation:
    """gp_likelihood.hpp:35-46 (+ telemetry)."""
    value: float = 0.0
    gradient: Optional[np.ndarray] = None
    solve_iterations: int = 0
    forward_gammas: Optional[np.ndarray] = None
    backward_gammas: Optional[np.ndarray] = None
    probe_seed: int = 0
    value_sample_variance: float = 0.0
    forward_cg_iterations: Optional[np.ndarray] = None
    total_cg_iterations: int = 0
    logdet: float = 0.0
    logdet_precond: float = 0.0
    quad: float = 0.0
    refine_passes: int = 0
    max_true_rel_residual: float = -1.0
    seconds_solve: float = 0.0
    seconds_backward: float = 0.0
    seconds_total: float = 0.0
    kernel_entries: int = 0
    mvm_flops: int = 0
    gpu_launches: int = 0
    max_cg_rel_residual: float = 0.0
    unconverged_columns: int = 0
    backward_mode_used: str = ""


def _result_struct(n_params, l):
    g = np.zeros(n_params)
    fg = np.zeros(l)
    bg = np.zeros((n_params, l))
    fi = np.zeros(l, dtype=np.int32)
    r = capi.gpk_mll_result()
    r.gradient = _ptr(g)
    r.forward_gammas = _ptr(fg)
    r.backward_gammas = _ptr(bg)
    r.forward_cg_iterations = fi.ctypes.data_as(C.POINTER(C.c_int))
    return r, (g, fg, bg, fi)


def _to_eval(r, arrs, seed, with_gradient):
    g, fg, bg, fi = arrs
    return MllEvaluation(value=r.value, gradient=g if with_gradient else None, solve_iterations=r.solve_iterations,
                         forward_gammas=fg, backward_gammas=bg if with_gradient else None, probe_seed=seed,
                         value_sample_variance=r.value_sample_variance, forward_cg_iterations=fi,
                         total_cg_iterations=r.total_cg_iterations, logdet=r.logdet, logdet_precond=r.logdet_precond,
                         quad=r.quad, refine_passes=r.refine_passes, max_true_rel_residual=r.max_true_rel_residual,
                         seconds_solve=r.seconds_solve, seconds_backward=r.seconds_backward,
                         seconds_total=r.seconds_total, kernel_entries=r.kernel_entries, mvm_flops=r.mvm_flops,
                         gpu_launches=r.gpu_launches, max_cg_rel_residual=r.max_cg_rel_residual,
                         unconverged_columns=r.unconverged_columns,
                         backward_mode_used=("fused", "faithful")[r.backward_mode_used] if with_gradient else "")


def evaluate_mll(y, k: KernelOperator, prec, batch: ProbeBatch, cfg: MllConfig, with_gradient: bool = True):
    """Forward (+ backward) pass of gp_likelihood.hpp:51-103 as one device evaluation."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    if y.ndim != 1 or y.shape[0] != k.rows():
        raise InputError("evaluate_mll: label length does not match operator")
    if prec is None or k.preconditioner is not prec:
        raise InputError("evaluate_mll: preconditioner is not attached to this operator")
    if with_gradient and isinstance(prec, DiagPlusLowRank) and prec.rank() > 0 and not prec.has_derivatives():
        raise InputError("DiagPlusLowRank: derivative factors not attached")
    z = np.asfortranarray(batch.probes, dtype=np.float64)
    if z.shape[0] != k.rows():
        raise InputError("vr_logdet: probe length does not match operator")
    l = z.shape[1]
    r, arrs = _result_struct(k.num_params(), l)
    cc = cfg.c(with_gradient)
    k.ctx.check(k.ctx.lib.gpk_evaluate_mll(k.ctx.h, _ptr(y), _ptr(z), z.shape[0], l, C.c_uint64(batch.seed),
                                           C.byref(cc), C.byref(r)))
    return _to_eval(r, arrs, batch.seed, with_gradient)


def evaluate_mll_device(y_dev, z_dev, k: KernelOperator, cfg: MllConfig, seed: int = 0, with_gradient=True):
    """Device-resident variant: y_dev (n,) and z_dev (l, n) are CUDA float64 buffers exposing data_ptr()
    (column-major n x l probes)."""
    n = k.rows()
    l = int(z_dev.shape[0])
    r, arrs = _result_struct(k.num_params(), l)
    cc = cfg.c(with_gradient)
    k.ctx.check(k.ctx.lib.gpk_evaluate_mll_device(k.ctx.h, C.c_void_p(y_dev.data_ptr()), C.c_void_p(z_dev.data_ptr()),
                                                  n, l, C.c_uint64(seed), C.byref(cc), C.byref(r)))
    return _to_eval(r, arrs, seed, with_gradient)


def mll_estimate(y, k, prec, batch, solver: CgConfig):
    """gp_likelihood.hpp:105-109"""
    return evaluate_mll(y, k, prec, batch, MllConfig(solver, True), with_gradient=False).value


def mll_gradient(y, k, prec, batch, solver: CgConfig):
    """gp_likelihood.hpp:111-115"""
    return evaluate_mll(y, k, prec, batch, MllConfig(solver, True), with_gradient=True).gradient


# ---------------------------------------------------------------------------
# the callers of the hot path — dense exact mLL (validation / test
# metric), cross-kernel predictive mean, and the optimize() step driver.
# ---------------------------------------------------------------------------
@dataclass
class ExactMll:
    """gp_likelihood.hpp:119-122"""
    value: float
    gradient: Optional[np.ndarray]


def mll_exact(y, x, spec: KernelSpec, params: Hyperparameters, with_gradient: bool = True, device: int = 0):
    """Dense exact mLL (+ log-space gradient) on the device (gp_likelihood.hpp:124-146)."""
    op = KernelOperator(spec, x, params, device=device)
    return op_mll_exact(op, y, with_gradient)


def op_mll_exact(op: KernelOperator, y, with_gradient: bool = True):
    y = np.ascontiguousarray(y, dtype=np.float64)
    if y.ndim != 1 or y.shape[0] != op.rows():
        raise InputError("mll_exact: label length does not match data")
    v = C.c_double()
    g = np.zeros(op.num_params()) if with_gradient else None
    op.ctx.check(op.ctx.lib.gpk_mll_exact(op.ctx.h, _ptr(y), C.byref(v), _ptr(g)))
    return ExactMll(v.value, g)


def cross_kernel_mvm(op: KernelOperator, a, v):
    """cross_kernel(spec, params, A, X) @ v (kernels.hpp:339-354), X = the operator's data."""
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2 or a.shape[1] != op.dim():
        raise InputError("cross_kernel: dimension mismatch")
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.shape != (op.rows(),):
        raise InputError("cross_kernel: dimension mismatch")
    out = np.empty(a.shape[0])
    op.ctx.check(op.ctx.lib.gpk_cross_kernel_mvm(op.ctx.h, _ptr(a), a.shape[0], a.shape[0], _ptr(v), _ptr(out)))
    return out


def predict_mean(op: KernelOperator, y, x_test, solver: CgConfig):
    """run_training_arm's predictive mean (experiments.hpp:403-414) with the attached
    preconditioner: returns (mean, CG iterations of the K_hat alpha = y solve)."""
    if op.preconditioner is None:
        raise InputError("predict_mean: no preconditioner attached")
    y = np.ascontiguousarray(y, dtype=np.float64)
    if y.shape != (op.rows(),):
        raise InputError("pcg_solve: rhs length does not match operator")
    a = np.asfortranarray(np.asarray(x_test, dtype=np.float64))
    if a.ndim != 2 or a.shape[1] != op.dim():
        raise InputError("cross_kernel: dimension mismatch")
    out = np.empty(a.shape[0])
    it = C.c_int()
    cc = solver.c()
    op.ctx.check(op.ctx.lib.gpk_predict_mean(op.ctx.h, _ptr(y), _ptr(a), a.shape[0], a.shape[0], C.byref(cc),
                                             _ptr(out), C.byref(it)))
    return out, it.value


@dataclass
class Dataset:
    """dataset.hpp:18-26 (features n x d, targets n)."""
    x: np.ndarray
    y: np.ndarray

    def size(self):
        return 0 if self.x is None else int(np.shape(self.x)[0])


@dataclass
class Standardizer:
    """dataset.hpp:87-101: training-split column statistics; exactly invertible transforms."""
    feature_mean: np.ndarray
    feature_std: np.ndarray
    target_mean: float = 0.0
    target_std: float = 1.0

    def transform_x(self, x):
        return (np.asarray(x, dtype=np.float64) - self.feature_mean) / self.feature_std

    def transform_y(self, y):
        return (np.asarray(y, dtype=np.float64) - self.target_mean) / self.target_std

    def invert_x(self, x):
        return np.asarray(x, dtype=np.float64) * self.feature_std + self.feature_mean

    def invert_y(self, y):
        return np.asarray(y, dtype=np.float64) * self.target_std + self.target_mean


@dataclass
class SplitFractions:
    """dataset.hpp:111-113"""
    train: float = 0.64
    validation: float = 0.16
    test: float = 0.20


@dataclass
class DataSplits:
    """dataset.hpp:103-109"""
    train: Dataset
    validation: Dataset
    test: Dataset
    stats: Standardizer
    standardized: bool
    feature_names: list
    target_name: str


def load_csv(path: str, target_column: str, standardize: bool = True, split: SplitFractions = SplitFractions(),
             seed: int = 0) -> DataSplits:
    """load_csv (dataset.hpp:155-242) through gpk_load_csv: header row, mt19937_64 shuffle,
    llround split, training-split standardisation.  Raises InputError with the reference's
    messages (non-numeric cell with row/column, constant column naming the column, ...)."""
    lib = capi.lib()
    h = C.c_void_p()
    err = C.create_string_buffer(1024)
    rc = lib.gpk_load_csv(str(path).encode(), str(target_column).encode(), int(bool(standardize)),
                          float(split.train), float(split.validation), float(split.test),
                          int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(h), err, len(err))
    if rc != capi.GPK_OK:
        raise _ERRS.get(rc, GpkError)(err.value.decode())
    try:
        parts = []
        d = C.c_int()
        for s in (0, 1, 2):
            n = C.c_int64()
            lib.gpk_dataset_shape(h, s, C.byref(n), C.byref(d))
            x = np.zeros((n.value, d.value), dtype=np.float64, order="F")
            y = np.zeros(n.value, dtype=np.float64)
            if n.value:
                lib.gpk_dataset_copy(h, s, _ptr(x), max(1, n.value), _ptr(y))
            parts.append(Dataset(x, y))
        st = C.c_int()
        fm = np.zeros(d.value)
        fs = np.ones(d.value)
        tm, ts = C.c_double(), C.c_double()
        lib.gpk_dataset_stats(h, C.byref(st), _ptr(fm), _ptr(fs), C.byref(tm), C.byref(ts))
        names = [lib.gpk_dataset_column_name(h, j).decode() for j in range(d.value)]
        target = lib.gpk_dataset_column_name(h, -1).decode()
        return DataSplits(parts[0], parts[1], parts[2], Standardizer(fm, fs, tm.value, ts.value), bool(st.value),
                          names, target)
    finally:
        lib.gpk_dataset_free(h)


@dataclass
class OptOptions:
    """optimizer.hpp:24-43"""
    method: str = "lbfgs"  # "lbfgs" | "adam"
    max_steps: int = 20
    lbfgs_memory: int = 10
    armijo_c1: float = 1e-4
    wolfe_c2: float = 0.9
    adam_lr: float = 0.1
    early_stop_patience: int = 3
    validation_fraction: float = 0.16
    grad_tol: float = 1e-8
    max_line_search: int = 20

    def c(self):
        m = {"lbfgs": capi.GPK_OPT_LBFGS, "adam": capi.GPK_OPT_ADAM}.get(self.method)
        if m is None:
            raise InputError("OptOptions: unknown method")
        return capi.gpk_opt_options(m, int(self.max_steps), int(self.lbfgs_memory), float(self.armijo_c1),
                                    float(self.wolfe_c2), float(self.adam_lr), int(self.early_stop_patience),
                                    float(self.grad_tol), int(self.max_line_search))


@dataclass
class PivotedCholeskyBuilder:
    """build_preconditioner's pivoted-Cholesky branch (experiments.hpp:30-68)."""
    rank: int
    diag_tol: float = 0.0


@dataclass
class IdentityBuilder:
    """The baseline arm's builder (experiments.hpp:470-471): IdentityPreconditioner."""
    rank: int = -1


@dataclass
class StepRecord:  # optimizer.hpp:52-66
    theta: np.ndarray
    objective: float
    validation_metric: float
    model_evaluations_cumulative: int
    wall_time_s: float
    accepted: bool
    step_length: float
    f_before: float
    dir_derivative_before: float
    dir_derivative_after: float


@dataclass
class EvalRecord:  # optimizer.hpp:45-50
    step: int
    f: float
    grad_norm: float


@dataclass
class OptTrace:  # optimizer.hpp:68-72
    steps: list
    evaluations: list


_STOP_MESSAGES = {capi.GPK_OPT_MAX_STEPS: "", capi.GPK_OPT_GRAD_TOL: "gradient norm below tolerance",
                  capi.GPK_OPT_LINE_SEARCH_FAILED: "line search failed after bounded bisection; step rejected",
                  capi.GPK_OPT_STOPPED: "stopped by callback"}


@dataclass
class OptimizeResult:
    """optimizer.hpp:356-361 (+ the MinimizeResult fields and GPU telemetry)."""
    best: Hyperparameters
    trace: OptTrace
    best_validation: float
    final_train_neg_mll_per_point: float
    final_objective: float
    minimizer_steps: int
    converged: bool
    message: str
    total_cg_iterations: int
    seconds_total: float


def count_model_evaluations(trace: OptTrace) -> int:
    """optimizer.hpp:74"""
    return len(trace.evaluations)


def optimize(train: Dataset, validation: Optional[Dataset], spec: KernelSpec, init: Hyperparameters,
             precond_builder, probe_count: int, opts: OptOptions, mll_cfg: MllConfig, seed: int,
             dense_limit: int = 4096, device: int = 0) -> OptimizeResult:
    """optimize() (optimizer.hpp:404-505) on the device path (gpk_optimize): L-BFGS / Adam on the
    negative mLL in log space, preconditioner rebuilt and probes redrawn at every step start."""
    x = np.asfortranarray(np.asarray(train.x, dtype=np.float64))
    if x.ndim != 2 or x.shape[0] < 1:
        raise InputError("optimize: empty training set")
    if init.dim() != x.shape[1]:
        raise InputError("optimize: hyperparameter dimension mismatch")
    n, d = x.shape
    ytr = np.ascontiguousarray(train.y, dtype=np.float64)
    op = KernelOperator(spec, x, init, device=device)
    vop = None
    yv = None
    if validation is not None and validation.size() > 0:
        vop = KernelOperator(spec, validation.x, init, device=device)
        yv = np.ascontiguousarray(validation.y, dtype=np.float64)
    ard = bool(spec.ard)
    npo = d + 2 if ard else 3
    ms = int(opts.max_steps)
    cap = ms * (int(opts.max_line_search) + 1)
    best = np.zeros(d + 2)
    th = np.zeros((ms, npo))
    arr = {k: np.zeros(ms) for k in ("obj", "val", "wall", "len", "fb", "ddb", "dda")}
    acc = np.zeros(ms, dtype=np.int32)
    sev = np.zeros(ms, dtype=np.int64)
    est = np.zeros(cap, dtype=np.int32)
    ef = np.zeros(cap)
    eg = np.zeros(cap)
    r = capi.gpk_opt_result()
    r.best_log_params = _ptr(best)
    r.step_theta = _ptr(th)
    r.step_objective, r.step_validation, r.step_wall_time = _ptr(arr["obj"]), _ptr(arr["val"]), _ptr(arr["wall"])
    r.step_length, r.step_f_before = _ptr(arr["len"]), _ptr(arr["fb"])
    r.step_dir_derivative_before, r.step_dir_derivative_after = _ptr(arr["ddb"]), _ptr(arr["dda"])
    r.step_accepted = acc.ctypes.data_as(C.POINTER(C.c_int))
    r.step_evaluations = sev.ctypes.data_as(C.POINTER(C.c_longlong))
    r.eval_capacity = cap
    r.eval_step = est.ctypes.data_as(C.POINTER(C.c_int))
    r.eval_f, r.eval_grad_norm = _ptr(ef), _ptr(eg)
    theta0 = np.ascontiguousarray(init.to_log_vector(), dtype=np.float64)
    oc = opts.c()
    mc = mll_cfg.c(True)
    rank = int(getattr(precond_builder, "rank", -1))
    diag_tol = float(getattr(precond_builder, "diag_tol", 0.0))
    op.ctx.check(op.ctx.lib.gpk_optimize(op.ctx.h, _ptr(ytr), vop.ctx.h if vop else None, _ptr(yv), spec.code,
                                         int(ard), _ptr(theta0), rank, diag_tol, int(probe_count), C.byref(oc),
                                         C.byref(mc), C.c_uint64(seed), int(dense_limit), C.byref(r)))
    steps = [StepRecord(th[s].copy(), arr["obj"][s], arr["val"][s], int(sev[s]), arr["wall"][s], bool(acc[s]),
                        arr["len"][s], arr["fb"][s], arr["ddb"][s], arr["dda"][s]) for s in range(r.n_steps)]
    evals = [EvalRecord(int(est[e]), float(ef[e]), float(eg[e])) for e in range(min(r.n_evaluations, cap))]
    return OptimizeResult(Hyperparameters.from_log_vector(best), OptTrace(steps, evals), r.best_validation,
                          r.final_train_neg_mll_per_point, r.final_objective, r.minimizer_steps, bool(r.converged),
                          _STOP_MESSAGES.get(r.stop_reason, ""), int(r.total_cg_iterations), r.seconds_total)


@dataclass
class TrainingRow:
    """experiments.hpp:360-372 (the per-arm row of run_training)."""
    steps: int
    model_evaluations: int
    wall_time_s: float
    train_neg_mll_per_point: float
    test_neg_mll_per_point: float
    test_rmse: float
    final_params: Hyperparameters


def run_training_arm(train: Dataset, validation: Optional[Dataset], test: Optional[Dataset], spec: KernelSpec,
                     init: Hyperparameters, precond_builder, probe_count: int, opts: OptOptions,
                     solver: CgConfig, seed: int, dense_limit: int = 4096, device: int = 0) -> TrainingRow:
    """detail::run_training_arm (experiments.hpp:388-418): optimize, then the dense test metric and
    the predictive-mean RMSE with the preconditioner rebuilt at the best hyperparameters."""
    res = optimize(train, validation, spec, init, precond_builder, probe_count, opts, MllConfig(solver, True),
                   seed, dense_limit, device)
    test_nll, rmse = 0.0, 0.0
    if test is not None and test.size() > 0:
        test_nll = -mll_exact(test.y, test.x, spec, res.best, with_gradient=False, device=device).value / test.size()
        op = KernelOperator(spec, train.x, res.best, device=device)
        if int(getattr(precond_builder, "rank", -1)) < 0:
            IdentityPreconditioner(op)
        else:
            pivoted_cholesky(op, precond_builder.rank, precond_builder.diag_tol)
        mean, _ = predict_mean(op, train.y, test.x, solver)
        rmse = float(np.sqrt(np.sum((mean - np.asarray(test.y)) ** 2) / test.size()))
    return TrainingRow(len(res.trace.steps), count_model_evaluations(res.trace),
                       res.trace.steps[-1].wall_time_s if res.trace.steps else 0.0,
                       res.final_train_neg_mll_per_point, test_nll, rmse, res.best)
