"""CPU oracle for the preconditioned mBCG hot path — TEST INFRASTRUCTURE ONLY.

ctypes bindings over ``liboracle.so`` (an Eigen-free C++20 restatement of
/root/reference/proj/include/gpkrylov, see ``gpkrylov_oracle.cpp``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker.
The product package ``paper_2107_00243_b200`` never imports it.

All matrices are column-major float64 (Eigen's default layout), passed as
numpy arrays in Fortran order.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_NAME = "liboracle_native.so" if os.environ.get("ORC_NATIVE") == "1" else "liboracle.so"
_LIB_PATH = os.path.join(_HERE, _LIB_NAME)

RBF, MATERN12, MATERN32, MATERN52, RATQUAD = 0, 1, 2, 3, 4
DENSE, MATRIX_FREE, CACHED = 0, 1, 2
FAMILIES = {"rbf": RBF, "matern12": MATERN12, "matern32": MATERN32, "matern52": MATERN52, "ratquad": RATQUAD}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # 1 input_error, 2 numerical_error, 3 solver_error


class InputError(OracleError):
    pass


class NumericalError(OracleError):
    pass


class SolverError(NumericalError):
    pass


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (g++, -O3, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
        os.path.join(_HERE, "gpkrylov_oracle.cpp")
    ):
        subprocess.run(["make", "-C", _HERE, "-B" if force else _LIB_NAME], check=True,
                       stdout=subprocess.DEVNULL)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_mix_seed.restype = C.c_uint64
        _lib.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    return _lib


_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_L = C.POINTER(C.c_int64)


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def _f(a):
    """Fortran-ordered float64 copy (column-major)."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _check(rc: int):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        cls = {1: InputError, 2: NumericalError, 3: SolverError}.get(rc, OracleError)
        raise cls(rc, msg)


def mix_seed(seed: int, salt: int) -> int:
    return int(lib().orc_mix_seed(C.c_uint64(seed), C.c_uint64(salt)))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def make_probes(n: int, count: int, seed: int) -> np.ndarray:
    out = np.empty((n, count), dtype=np.float64, order="F")
    _check(lib().orc_make_probes(C.c_int64(n), C.c_int(count), C.c_uint64(seed), _p(out)))
    return out


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """proj/tests/support.hpp:13-19 — row-major draw order, mt19937_64 + normal_distribution."""
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    _check(lib().orc_random_matrix(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), _p(out)))
    return out


class Params:
    """Hyperparameters in log space (kernels.hpp:17-64)."""

    def __init__(self, d: int, outputscale=1.0, lengthscale=1.0, noise=1e-2, lengthscales=None):
        self.log_o = float(np.log(outputscale))
        ls = np.full(d, lengthscale, dtype=np.float64) if lengthscales is None else np.asarray(lengthscales, float)
        self.log_ls = np.ascontiguousarray(np.log(ls))
        self.log_noise = float(np.log(noise))

    @property
    def d(self):
        return len(self.log_ls)

    def raw(self, w):
        if w == 0:
            return float(np.exp(self.log_o))
        if 1 <= w <= self.d:
            return float(np.exp(self.log_ls[w - 1]))
        return float(np.exp(self.log_noise))


def kernel_apply(family, x, p: Params, v, which=-1, mode=MATRIX_FREE, block_rows=1024, alpha=1.0):
    x = _f(x)
    v = _f(v if np.ndim(v) == 2 else np.asarray(v)[:, None])
    n, d = x.shape
    out = np.empty_like(v, order="F")
    _check(lib().orc_kernel_apply(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                  C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), C.c_int(mode),
                                  C.c_int64(block_rows), C.c_int(which), _p(v), C.c_int(v.shape[1]), _p(out)))
    return out


def kernel_apply_block(family, x, p: Params, v, mode=CACHED, alpha=1.0):
    """KernelOperator::apply_block over all columns of v (oracle-internal block apply)."""
    x = _f(x)
    v = _f(v)
    n, d = x.shape
    out = np.empty_like(v, order="F")
    _check(lib().orc_kernel_apply_block(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                        C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), C.c_int(mode),
                                        _p(v), C.c_int(v.shape[1]), _p(out)))
    return out


def kernel_apply_rows(family, x, p: Params, rows, v, alpha=1.0):
    """Rows ``rows`` of (K + sigma^2 I) V with the MatrixFree entries and sums (kernels.hpp:184-195,
    :296-306): a (len(rows), t) array.  For MVM row-subset parity at the large BASELINE shapes."""
    x = _f(x)
    v = _f(v if np.ndim(v) == 2 else np.asarray(v)[:, None])
    n, d = x.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty((len(rows), v.shape[1]), order="F")
    _check(lib().orc_kernel_apply_rows(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                       C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise),
                                       rows.ctypes.data_as(_L), C.c_int64(len(rows)), _p(v), C.c_int(v.shape[1]),
                                       _p(out)))
    return out


def kernel_apply_parallel(family, x, p: Params, v, block_rows=1024, alpha=1.0):
    x = _f(x)
    v = _f(v)
    n, d = x.shape
    out = np.empty_like(v, order="F")
    _check(lib().orc_kernel_apply_parallel(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                           C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise),
                                           C.c_int64(block_rows), _p(v), C.c_int(v.shape[1]), _p(out)))
    return out


def kernel_column(family, x, p: Params, i, which=-1, alpha=1.0):
    x = _f(x)
    n, d = x.shape
    out = np.empty(n)
    _check(lib().orc_kernel_column(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                   C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), C.c_int(which),
                                   C.c_int64(i), _p(out)))
    return out


def dense(family, x, p: Params, which=-1, alpha=1.0):
    """Dense K_hat (which < 0) or dK_hat/dtheta_which (kernels.hpp:270-282)."""
    x = _f(x)
    n, d = x.shape
    out = np.empty((n, n), order="F")
    _check(lib().orc_dense(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                           C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), C.c_int(which), _p(out)))
    return out


def pcg_dense(a, b, prec="identity", pmat=None, noise=0.0, lfac=None, max_iters=100, rel_tol=1e-6,
              collect=False):
    """pcg_solve (krylov.hpp:47-129) on a dense SPD matrix."""
    a = _f(a)
    n = a.shape[0]
    b = np.ascontiguousarray(b, dtype=np.float64)
    kind = {"identity": 0, "exact": 1, "dplr": 2}[prec]
    pm = _f(pmat) if pmat is not None else None
    lf = _f(lfac) if lfac is not None else None
    k = lf.shape[1] if lf is not None else 0
    x = np.empty(n)
    it, cv = C.c_int(), C.c_int()
    td, ts, rh = np.zeros(max_iters), np.zeros(max_iters), np.zeros(max_iters)
    _check(lib().orc_pcg_dense(_p(a), C.c_int64(n), _p(b), C.c_int(kind), _p(pm), C.c_double(noise), _p(lf),
                               C.c_int64(k), C.c_int(max_iters), C.c_double(rel_tol), C.c_int(int(collect)), _p(x),
                               C.byref(it), C.byref(cv), _p(td), _p(ts), _p(rh)))
    m = it.value
    return dict(solution=x, iterations=m, converged=bool(cv.value), residual_history=rh[:m].copy(),
                tdiag=td[:m].copy() if collect else None, tsub=ts[: max(m - 1, 0)].copy() if collect else None)


def pcg_kernel(family, x, p: Params, b, rank=-1, max_iters=100, rel_tol=1e-6, alpha=1.0):
    """batched pcg_solve on the MatrixFree kernel operator, pivoted-Cholesky(rank) or identity (rank<0)."""
    x = _f(x)
    b = _f(b if np.ndim(b) == 2 else np.asarray(b)[:, None])
    n, d = x.shape
    t = b.shape[1]
    sol = np.empty_like(b, order="F")
    iters = np.zeros(t, dtype=np.int32)
    conv = np.zeros(t, dtype=np.int32)
    _check(lib().orc_pcg_kernel(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), C.c_int(rank), _p(b),
                                C.c_int(t), C.c_int(max_iters), C.c_double(rel_tol), _p(sol),
                                iters.ctypes.data_as(_I), conv.ctypes.data_as(_I)))
    return sol, iters, conv


def slq(diag, sub, clamp_floor=None):
    """slq_quadrature with f = log (trace_estimation.hpp:88-110)."""
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    sub = np.ascontiguousarray(sub, dtype=np.float64)
    m = len(diag)
    val = C.c_double()
    nodes, weights = np.zeros(m), np.zeros(m)
    cl = C.c_int()
    _check(lib().orc_slq(_p(diag), _p(sub), C.c_int(m), C.c_double(clamp_floor or 0.0),
                         C.c_int(clamp_floor is not None), C.byref(val), _p(nodes), _p(weights), C.byref(cl)))
    return dict(value=val.value, nodes=nodes, weights=weights, clamped=cl.value)


def pivoted_cholesky(rank, diag_tol=0.0, kmat=None, family=RBF, x=None, p: Params | None = None, alpha=1.0):
    """preconditioners.hpp:236-264 over a dense matrix (kmat) or the kernel operator."""
    if kmat is not None:
        km = _f(kmat)
        n, d = km.shape[0], 0
        xx = None
        lo, ll, ln = 0.0, None, 0.0
    else:
        xx = _f(x)
        n, d = xx.shape
        km = None
        lo, ll, ln = p.log_o, p.log_ls, p.log_noise
    lout = np.zeros((n, max(rank, 0)), order="F")
    piv = np.zeros(max(rank, 1), dtype=np.int64)
    ach = C.c_int()
    rem = np.zeros(n)
    _check(lib().orc_pivoted_cholesky(_p(km), C.c_int(family), C.c_double(alpha), _p(xx), C.c_int64(n), C.c_int(d),
                                      C.c_double(lo), _p(ll), C.c_double(ln), C.c_int(rank), C.c_double(diag_tol),
                                      _p(lout), piv.ctypes.data_as(_L), C.byref(ach), _p(rem)))
    k = ach.value
    return dict(L=np.asfortranarray(lout.reshape(-1, order="F")[: n * k].reshape((n, k), order="F")),
                pivots=piv[:k].copy(), rank=k, remaining=rem)


def deriv_factors(family, x, p: Params, L, pivots, alpha=1.0):
    """pivoted_cholesky_deriv_factors (preconditioners.hpp:269-295): list of d+2 n x k arrays."""
    x = _f(x)
    L = _f(L)
    n, d = x.shape
    k = L.shape[1]
    out = np.zeros((d + 2, n, k))
    buf = np.zeros((d + 2) * n * k)
    piv = np.ascontiguousarray(pivots, dtype=np.int64)
    _check(lib().orc_deriv_factors(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                   C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), _p(L),
                                   piv.ctypes.data_as(_L), C.c_int(k), _p(buf)))
    for w in range(d + 2):
        out[w] = buf[w * n * k:(w + 1) * n * k].reshape((n, k), order="F")
    return out


def dplr(noise, L, v):
    """DiagPlusLowRank solve / apply / logdet / tr(P^{-1}) (preconditioners.hpp:82-186)."""
    L = _f(L)
    n, k = L.shape
    v = np.ascontiguousarray(v, dtype=np.float64)
    s, a = np.empty(n), np.empty(n)
    ld, tr = C.c_double(), C.c_double()
    _check(lib().orc_dplr(C.c_double(noise), _p(L), C.c_int64(n), C.c_int64(k), _p(v), _p(s), _p(a), C.byref(ld),
                          C.byref(tr)))
    return dict(solve=s, apply=a, logdet=ld.value, trace_inv=tr.value)


def dplr_trace_inv_deriv(noise, L, dL, shift=0.0):
    L = _f(L)
    dL = _f(dL)
    n, k = L.shape
    out = C.c_double()
    _check(lib().orc_dplr_trace_inv_deriv(C.c_double(noise), _p(L), _p(dL), C.c_int64(n), C.c_int64(k),
                                          C.c_double(shift), C.byref(out)))
    return out.value


def evaluate_mll(family, x, p: Params, y, probes, seed=0, prec="pivchol", rank=0, diag_tol=0.0, mode=MATRIX_FREE,
                 max_iters=100, rel_tol=1e-6, share_probes=True, with_gradient=True, alpha=1.0, lockstep=False):
    """evaluate_mll (gp_likelihood.hpp:51-103) with the preconditioner built as
    build_preconditioner's pivoted-Cholesky branch (experiments.hpp:37-38, :59-61).

    ``lockstep=True`` runs every solve of a phase as one lock-step batch (the batched_pcg
    contract, krylov.hpp:131-153); with ``mode=CACHED`` the operator keeps its MatrixFree
    kernel block and applies it to the whole block per iteration — bitwise the MatrixFree
    per-column result (tests/test_oracle_lockstep.py), fast enough for the C2 fixtures."""
    x = _f(x)
    n, d = x.shape
    z = _f(probes)
    l = z.shape[1]
    y = np.ascontiguousarray(y, dtype=np.float64)
    kind = {"identity": 0, "pivchol": 1, "exact": 2}[prec]
    grad = np.zeros(d + 2)
    fg = np.zeros(l)
    bg = np.zeros((d + 2) * l)
    fi = np.zeros(l, dtype=np.int32)
    sc = np.zeros(8)
    u = np.zeros(n)
    piv = np.zeros(max(rank, 1), dtype=np.int64)
    _check(lib().orc_evaluate_mll2(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                   C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), _p(y), _p(z),
                                   C.c_int(l), C.c_uint64(seed), C.c_int(kind), C.c_int(rank), C.c_double(diag_tol),
                                   C.c_int(mode), C.c_int(max_iters), C.c_double(rel_tol), C.c_int(int(share_probes)),
                                   C.c_int(int(with_gradient)), C.c_int(int(lockstep)), _p(grad), _p(fg), _p(bg),
                                   fi.ctypes.data_as(_I), _p(sc), _p(u), piv.ctypes.data_as(_L)))
    return dict(value=sc[0], logdet=sc[1], quad=sc[2], value_sample_variance=sc[3], solve_iterations=int(sc[4]),
                total_cg_iterations=int(sc[5]), logdet_precond=sc[6], gradient=grad, forward_gammas=fg,
                backward_gammas=bg.reshape(d + 2, l), forward_cg_iterations=fi, u=u,
                pivots=piv[:rank].copy() if kind == 1 else None)


def mll_exact(family, x, p: Params, y, alpha=1.0):
    """mll_exact (gp_likelihood.hpp:124-146)."""
    x = _f(x)
    n, d = x.shape
    y = np.ascontiguousarray(y, dtype=np.float64)
    val = C.c_double()
    grad = np.zeros(d + 2)
    _check(lib().orc_mll_exact(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                               C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), _p(y), C.byref(val),
                               _p(grad)))
    return val.value, grad


def dense_spd(a, want_log=False):
    """oracle.hpp dual routes: (logdet_chol, logdet_eig, eigvals, matlog)."""
    a = _f(a)
    n = a.shape[0]
    lc, le = C.c_double(), C.c_double()
    ev = np.zeros(n)
    ml = np.zeros((n, n), order="F") if want_log else None
    _check(lib().orc_dense_spd(_p(a), C.c_int64(n), C.byref(lc), C.byref(le), _p(ev), _p(ml)))
    return lc.value, le.value, ev, ml


# ---------------------------------------------------------------------------
# the callers of the hot path
# ---------------------------------------------------------------------------
def mll_exact_value(family, x, p: Params, y, alpha=1.0):
    """mll_exact(...).value (gp_likelihood.hpp:124-146) without the O(n^3) gradient."""
    x = _f(x)
    n, d = x.shape
    y = np.ascontiguousarray(y, dtype=np.float64)
    val = C.c_double()
    _check(lib().orc_mll_exact_value(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d),
                                     C.c_double(p.log_o), _p(p.log_ls), C.c_double(p.log_noise), _p(y),
                                     C.byref(val)))
    return val.value


def cross_kernel_mvm(family, a, b, p: Params, v, alpha=1.0):
    """cross_kernel(spec, params, A, B) @ v (kernels.hpp:339-354)."""
    a, b = _f(a), _f(b)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty(a.shape[0])
    _check(lib().orc_cross_kernel_mvm(C.c_int(family), C.c_double(alpha), _p(a), C.c_int64(a.shape[0]), _p(b),
                                      C.c_int64(b.shape[0]), C.c_int(a.shape[1]), C.c_double(p.log_o),
                                      _p(p.log_ls), C.c_double(p.log_noise), _p(v), _p(out)))
    return out


def predict_mean(family, x, y, xs, p: Params, rank=-1, diag_tol=0.0, dense_limit=4096, max_iters=100,
                 rel_tol=1e-6, alpha=1.0):
    """run_training_arm's predictive mean (experiments.hpp:403-414). Returns (mean, cg iterations)."""
    x, xs = _f(x), _f(xs)
    n, d = x.shape
    y = np.ascontiguousarray(y, dtype=np.float64)
    mean = np.empty(xs.shape[0])
    it = C.c_int()
    _check(lib().orc_predict_mean(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d), _p(y),
                                  _p(xs), C.c_int64(xs.shape[0]), C.c_double(p.log_o), _p(p.log_ls),
                                  C.c_double(p.log_noise), C.c_int(rank), C.c_double(diag_tol),
                                  C.c_int64(dense_limit), C.c_int(max_iters), C.c_double(rel_tol), _p(mean),
                                  C.byref(it)))
    return mean, it.value


OPT_DEFAULTS = dict(method=0, max_steps=20, lbfgs_memory=10, armijo_c1=1e-4, wolfe_c2=0.9, adam_lr=0.1,
                    early_stop_patience=3, grad_tol=1e-8, max_line_search=20)


def optimize(family, x, y, xv, yv, p0: Params, ard=True, rank=0, diag_tol=0.0, probe_count=8, max_iters=100,
             rel_tol=1e-6, share_probes=True, seed=17, dense_limit=4096, alpha=1.0, **opts):
    """optimize() (optimizer.hpp:404-505) with the pivoted-Cholesky builder (rank >= 0) or the
    identity (rank < 0), per-step probe rotation mix_seed(seed, step) and early stopping."""
    o = dict(OPT_DEFAULTS, **opts)
    x = _f(x)
    n, d = x.shape
    y = np.ascontiguousarray(y, dtype=np.float64)
    nv = 0 if xv is None else int(np.shape(xv)[0])
    xvf = _f(xv) if nv else None
    yvf = np.ascontiguousarray(yv, dtype=np.float64) if nv else None
    theta0 = np.concatenate([[p0.log_o], p0.log_ls, [p0.log_noise]])
    optv = np.array([o["method"], o["max_steps"], o["lbfgs_memory"], o["armijo_c1"], o["wolfe_c2"], o["adam_lr"],
                     o["early_stop_patience"], o["grad_tol"], o["max_line_search"]], dtype=np.float64)
    ms = int(o["max_steps"])
    npo = d + 2 if ard else 3
    cap = ms * (int(o["max_line_search"]) + 1)
    best = np.zeros(d + 2)
    sc = np.zeros(8)
    rows = np.zeros((ms, 8))
    th = np.zeros((ms, npo))
    ev = np.zeros((cap, 3))
    _check(lib().orc_optimize(C.c_int(family), C.c_double(alpha), _p(x), C.c_int64(n), C.c_int(d), _p(y), _p(xvf),
                              C.c_int64(nv), _p(yvf), C.c_int(int(ard)), _p(theta0), C.c_int(rank),
                              C.c_double(diag_tol), C.c_int(probe_count), _p(optv), C.c_int(max_iters),
                              C.c_double(rel_tol), C.c_int(int(share_probes)), C.c_uint64(seed),
                              C.c_int64(dense_limit), _p(best), _p(sc), _p(rows), _p(th), _p(ev), C.c_int(cap)))
    ns, ne = int(sc[5]), int(sc[6])
    return dict(best=best, best_validation=sc[0], final_train_neg_mll_per_point=sc[1], final_objective=sc[2],
                converged=bool(sc[3]), stop_reason=int(sc[4]), minimizer_steps=int(sc[7]),
                steps=[dict(theta=th[s].copy(), objective=rows[s, 0], validation_metric=rows[s, 1],
                            step_length=rows[s, 2], f_before=rows[s, 3], dir_derivative_before=rows[s, 4],
                            dir_derivative_after=rows[s, 5], accepted=bool(rows[s, 6]),
                            model_evaluations_cumulative=int(rows[s, 7])) for s in range(ns)],
                evaluations=[dict(step=int(ev[e, 0]), f=ev[e, 1], grad_norm=ev[e, 2]) for e in range(min(ne, cap))])


def minimize_quadratic(xstar, x0, method=0, max_steps=20, lbfgs_memory=10, armijo_c1=1e-4, wolfe_c2=0.9,
                       adam_lr=0.1, grad_tol=1e-8, max_line_search=20):
    """the optimizer.hpp minimizers on f = 0.5 |x - x*|^2 (GP bypassed)."""
    xstar = np.ascontiguousarray(xstar, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    m = xstar.size
    opt = np.array([max_steps, lbfgs_memory, armijo_c1, wolfe_c2, adam_lr, grad_tol, max_line_search], float)
    traj = np.zeros((max_steps + 1, m))
    certs = np.zeros((max_steps, 4))
    sc = np.zeros(3)
    _check(lib().orc_minimize_quadratic(C.c_int(method), C.c_int(m), _p(xstar), _p(x0), _p(opt), _p(traj),
                                        _p(certs), _p(sc)))
    ns = int(sc[0])
    return dict(trajectory=traj[: ns + 1].copy(), certificates=certs[:ns].copy(), steps=ns, evaluations=int(sc[1]),
                reason=int(sc[2]))
