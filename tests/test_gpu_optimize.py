"""GPU parity of the hot path's callers against the oracle:
the device dense mll_exact (gp_likelihood.hpp:124-146), the cross-kernel MVM
(kernels.hpp:339-354), the predictive mean (experiments.hpp:403-414) and the
optimize() step driver (optimizer.hpp:404-505, gpk_optimize) — trajectories,
evaluation counts, stop reasons and best iterates on identical data, probes
and seeds."""
import numpy as np
import pytest

import paper_2107_00243_b200 as gk
from paper_2107_00243_b200 import gpkrylov

pytestmark = pytest.mark.gpu

FAM = {0: "rbf", 1: "matern12", 2: "matern32", 3: "matern52"}


def gp_problem(orc, n, nv, d, fam, ls, noise, seed):
    x = orc.random_matrix(n + nv, d, seed)
    p = orc.Params(d, 1.0, ls, noise)
    K = orc.dense(fam, x, p)
    y = np.linalg.cholesky(K) @ orc.random_matrix(n + nv, 1, seed + 1)[:, 0]
    return x[:n], y[:n], x[n:], y[n:]


def hp(p):
    return gk.Hyperparameters(p.log_o, np.array(p.log_ls), p.log_noise)


@pytest.mark.parametrize("fam", [0, 1, 2, 3])
def test_mll_exact_matches_oracle(orc, fam):
    x, y, _, _ = gp_problem(orc, 300, 0, 3, fam, 0.9, 0.03, 3 + fam)
    p = orc.Params(3, 1.1, 0.8, 0.02, lengthscales=[0.6, 0.9, 1.3])
    want_v, want_g = orc.mll_exact(fam, x, p, y)
    got = gpkrylov.mll_exact(y, x, gk.KernelSpec(FAM[fam]), hp(p))
    assert got.value == pytest.approx(want_v, rel=1e-10)
    assert np.allclose(got.gradient, want_g, rtol=1e-8, atol=1e-8 * np.abs(want_g).max())
    v2 = gpkrylov.mll_exact(y, x, gk.KernelSpec(FAM[fam]), hp(p), with_gradient=False)
    assert v2.value == pytest.approx(want_v, rel=1e-12) and v2.gradient is None


def test_mll_exact_not_pd_raises(orc):
    x = np.zeros((10, 1))  # all-equal inputs: K = o^2 11^T, not PD with a tiny noise
    y = np.ones(10)
    with pytest.raises(gk.NumericalError, match="Cholesky factorization failed"):
        gpkrylov.mll_exact(y, x, gk.KernelSpec("rbf"), gk.Hyperparameters.from_raw(1, 1.0, 1.0, 1e-300))


@pytest.mark.parametrize("fam", [0, 1, 2, 3])
def test_cross_kernel_mvm_matches_oracle(orc, fam):
    a = orc.random_matrix(333, 5, 40)
    b = orc.random_matrix(1000, 5, 41)
    p = orc.Params(5, 1.3, 0.9, 0.05)
    v = orc.random_matrix(1000, 1, 42)[:, 0]
    want = orc.cross_kernel_mvm(fam, a, b, p, v)
    op = gk.KernelOperator(gk.KernelSpec(FAM[fam]), b, hp(p))
    got = gpkrylov.cross_kernel_mvm(op, a, v)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


@pytest.mark.parametrize("rank", [-1, 16])
def test_predict_mean_matches_oracle(orc, rank):
    x, y, xs, _ = gp_problem(orc, 600, 90, 2, orc.MATERN32, 0.7, 0.02, 21)
    p = orc.Params(2, 1.0, 0.7, 0.02)
    want, _ = orc.predict_mean(orc.MATERN32, x, y, xs, p, rank=rank, max_iters=2000, rel_tol=1e-11)
    op = gk.KernelOperator(gk.KernelSpec("matern32"), x, hp(p))
    if rank < 0:
        gk.IdentityPreconditioner(op)
    else:
        gk.pivoted_cholesky(op, rank)
    for prec, tol in (("fp64", 1e-8), ("tf32x3", 1e-5)):
        got, it = gpkrylov.predict_mean(op, y, xs, gk.CgConfig(2000, 1e-11 if prec == "fp64" else 1e-7, False,
                                                                prec, 3))
        assert it > 0
        assert np.linalg.norm(got - want) <= tol * np.linalg.norm(want), prec


def run_both(orc, x, y, xv, yv, p0, fam=0, ard=True, rank=8, probes=8, dense_limit=4096, max_iters=500,
             rel_tol=1e-10, **opts):
    want = orc.optimize(fam, x, y, xv, yv, p0, ard=ard, rank=rank, probe_count=probes, max_iters=max_iters,
                        rel_tol=rel_tol, seed=17, dense_limit=dense_limit, **opts)
    o = gpkrylov.OptOptions(method="adam" if opts.get("method", 0) == 1 else "lbfgs",
                            max_steps=opts.get("max_steps", 20), max_line_search=opts.get("max_line_search", 20),
                            adam_lr=opts.get("adam_lr", 0.1))
    builder = gpkrylov.IdentityBuilder() if rank < 0 else gpkrylov.PivotedCholeskyBuilder(rank)
    got = gpkrylov.optimize(gpkrylov.Dataset(x, y), gpkrylov.Dataset(xv, yv) if xv is not None else None,
                            gk.KernelSpec(FAM[fam], ard=ard), hp(p0), builder, probes, o,
                            gk.MllConfig(gk.CgConfig(max_iters, rel_tol, False, "fp64", 0)), 17, dense_limit)
    return want, got


def assert_same_run(want, got, tol=1e-6):
    assert len(got.trace.evaluations) == len(want["evaluations"])
    assert len(got.trace.steps) == len(want["steps"])
    for gs, ws in zip(got.trace.steps, want["steps"]):
        assert gs.accepted == ws["accepted"]
        assert gs.model_evaluations_cumulative == ws["model_evaluations_cumulative"]
        assert np.allclose(gs.theta, ws["theta"], rtol=tol, atol=tol)
        assert gs.objective == pytest.approx(ws["objective"], rel=tol)
        assert gs.validation_metric == pytest.approx(ws["validation_metric"], rel=tol, abs=tol)
    for ge, we in zip(got.trace.evaluations, want["evaluations"]):
        assert ge.step == we["step"]
        # trial points of a first unit step can land at overflowing hyperparameters where
        # the operator is numerically singular: there one arithmetic breaks down (+inf) and
        # the other returns a huge value; both reject the trial identically
        degenerate = not np.isfinite(we["f"]) or not np.isfinite(ge.f) or we["grad_norm"] > 1e8
        if not degenerate:
            assert ge.f == pytest.approx(we["f"], rel=tol)
            assert ge.grad_norm == pytest.approx(we["grad_norm"], rel=1e-4)
    assert np.allclose(got.best.to_log_vector(), want["best"], rtol=tol, atol=tol)
    assert got.final_train_neg_mll_per_point == pytest.approx(want["final_train_neg_mll_per_point"], rel=tol)


def test_optimize_lbfgs_matches_oracle(orc):
    x, y, xv, yv = gp_problem(orc, 120, 40, 2, orc.RBF, 0.8, 0.05, 5)
    want, got = run_both(orc, x, y, xv, yv, orc.Params(2, 1.0, 1.0, 0.01), max_steps=8, max_line_search=60)
    assert sum(s["accepted"] for s in want["steps"]) >= 2
    assert_same_run(want, got)
    assert got.message == {0: "", 1: "gradient norm below tolerance",
                           2: "line search failed after bounded bisection; step rejected",
                           3: "stopped by callback"}[want["stop_reason"]]
    assert got.total_cg_iterations > 0


def test_optimize_lbfgs_failed_line_search_matches_oracle(orc):
    x, y, xv, yv = gp_problem(orc, 120, 40, 2, orc.RBF, 0.8, 0.05, 5)
    want, got = run_both(orc, x, y, xv, yv, orc.Params(2, 1.0, 1.0, 0.01), max_steps=4, max_line_search=3)
    assert want["stop_reason"] == 2
    assert_same_run(want, got)
    assert got.message.startswith("line search failed")


def test_optimize_adam_isotropic_identity_matches_oracle(orc):
    x, y, xv, yv = gp_problem(orc, 150, 50, 3, orc.MATERN52, 0.9, 0.05, 8)
    want, got = run_both(orc, x, y, xv, yv, orc.Params(3, 1.0, 1.0, 0.01), fam=3, ard=False, rank=-1, method=1,
                         max_steps=6)
    assert_same_run(want, got)
    assert len(got.trace.steps[0].theta) == 3


def test_optimize_matrix_free_validation_path_matches_oracle(orc):
    # validation set above dense_limit: the identity-preconditioned value-only estimate with
    # probes mix_seed(seed, 0x7a11) (optimizer.hpp:464-470); training metric = f / n
    x, y, xv, yv = gp_problem(orc, 100, 60, 2, orc.MATERN32, 0.8, 0.05, 9)
    want, got = run_both(orc, x, y, xv, yv, orc.Params(2, 1.0, 0.8, 0.04), fam=2, method=1, max_steps=4,
                         dense_limit=50)
    assert all(s["validation_metric"] != 0.0 for s in want["steps"])
    assert_same_run(want, got)


def test_optimize_deterministic_and_no_validation(orc):
    x, y, _, _ = gp_problem(orc, 100, 0, 2, orc.RBF, 0.8, 0.05, 12)
    p0 = orc.Params(2, 1.0, 0.8, 0.04)
    want, a = run_both(orc, x, y, None, None, p0, method=1, max_steps=3)
    _, b = run_both(orc, x, y, None, None, p0, method=1, max_steps=3)
    assert a.best_validation == np.inf
    assert np.array_equal(a.best.to_log_vector(), b.best.to_log_vector())
    assert [e.f for e in a.trace.evaluations] == [e.f for e in b.trace.evaluations]
    assert_same_run(want, a)


def test_optimize_input_errors(orc):
    x = orc.random_matrix(20, 2, 1)
    y = np.zeros(20)
    with pytest.raises(gk.InputError, match="c1 < c2"):
        gpkrylov.optimize(gpkrylov.Dataset(x, y), None, gk.KernelSpec("rbf"), gk.Hyperparameters.from_raw(2),
                          gpkrylov.IdentityBuilder(), 4, gpkrylov.OptOptions(wolfe_c2=1e-5), gk.MllConfig(), 1)
    with pytest.raises(gk.InputError, match="dimension mismatch"):
        gpkrylov.optimize(gpkrylov.Dataset(x, y), None, gk.KernelSpec("rbf"), gk.Hyperparameters.from_raw(3),
                          gpkrylov.IdentityBuilder(), 4, gpkrylov.OptOptions(), gk.MllConfig(), 1)


def test_run_training_arm_end_to_end(orc):
    # SPEC.md:628 scaled: n = 500 1-d RBF GP; the identity arm's final train -L within
    # 1e-2 nats / point of the dense-oracle L-BFGS run; test RMSE of the predictive mean
    x, y, xv, yv = gp_problem(orc, 500, 100, 1, orc.RBF, 0.5, 0.01, 11)
    xs, ys = xv[:50], yv[:50]
    xv, yv = xv[50:], yv[50:]
    p0 = orc.Params(1, 1.0, 1.0, 0.01)
    dense = orc.optimize(orc.RBF, x, y, xv, yv, p0, rank=-2, probe_count=8, max_iters=500)
    row = gpkrylov.run_training_arm(gpkrylov.Dataset(x, y), gpkrylov.Dataset(xv, yv), gpkrylov.Dataset(xs, ys),
                                    gk.KernelSpec("rbf"), hp(p0), gpkrylov.IdentityBuilder(), 8,
                                    gpkrylov.OptOptions(), gk.CgConfig(500, 1e-6, False, "tf32x3", 2), 17)
    assert abs(row.train_neg_mll_per_point - dense["final_train_neg_mll_per_point"]) <= 1e-2
    assert row.steps >= 1 and row.model_evaluations >= row.steps
    assert row.test_rmse < 0.3
    assert np.isfinite(row.test_neg_mll_per_point)
