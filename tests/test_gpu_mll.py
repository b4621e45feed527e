"""GPU parity of the batched solver and of evaluate_mll against the oracle
(live on small seeded problems, and against the committed golden fixtures at
the BASELINE C1 workload)."""
import json
import math
import os

import numpy as np
import pytest

import paper_2107_00243_b200 as gk
from paper_2107_00243_b200 import workloads

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def make_op(fam, x, p, d):
    return gk.KernelOperator(gk.KernelSpec(fam), x, gk.Hyperparameters(p.log_o, np.array(p.log_ls), p.log_noise))


# ---------------------------------------------------------------------------
# batched solver (krylov.hpp)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("rank", [-1, 0, 8])
def test_mbcg_fp64_matches_oracle_pcg(orc, rank):
    n, d = 400, 2
    x = orc.random_matrix(n, d, 26)
    p = orc.Params(d, 1.0, 0.7, 0.05)
    b = orc.random_matrix(n, 6, 260)
    want, wit, wcv = orc.pcg_kernel(orc.RBF, x, p, b, rank=rank, max_iters=300, rel_tol=1e-8)
    op = make_op("rbf", x, p, d)
    prec = gk.IdentityPreconditioner(op) if rank < 0 else gk.pivoted_cholesky(op, rank)
    res = gk.batched_pcg(op, b, prec, gk.CgConfig(300, 1e-8, True, "fp64", 0))
    for c in range(6):
        # unpreconditioned CG (kappa ~ 1e5 here) loses orthogonality, so iteration counts at
        # tol 1e-8 drift with last-bit rounding; the solutions still agree to the tolerance
        # (rank 0 is P = sigma^2 I: the same iterates as plain CG; kappa is still ~1e4 at rank 8)
        slack = max(1, int(0.05 * wit[c])) if rank > 0 else max(1, int(0.1 * wit[c]))
        assert abs(res[c].iterations_used - wit[c]) <= slack
        assert res[c].converged == bool(wcv[c])
        assert rel(res[c].solution, want[:, c]) < (1e-7 if rank > 0 else 1e-5)


def test_mbcg_tridiagonal_matches_oracle(orc):
    n = 300
    x = orc.random_matrix(n, 1, 61)
    p = orc.Params(1, 1.0, 0.4, 0.05)
    k = orc.dense(orc.RBF, x, p)
    z = orc.make_probes(n, 1, 99)[:, 0]
    want = orc.pcg_dense(k, z, max_iters=40, rel_tol=1e-10, collect=True)
    op = make_op("rbf", x, p, 1)
    r = gk.pcg_solve(op, z, gk.IdentityPreconditioner(op), gk.CgConfig(40, 1e-10, True, "fp64", 0))
    # Plain CG on this kernel (kappa ~ 6e3) loses orthogonality after a few steps, from which point
    # the T entries of two correct fp64 implementations diverge with last-bit rounding; the leading
    # entries and the Gauss quadrature (the SLQ value the estimator uses) agree.
    assert abs(r.iterations_used - want["iterations"]) <= max(1, int(0.1 * want["iterations"]))
    m0 = 6
    assert np.allclose(r.tridiag.diag[:m0], want["tdiag"][:m0], rtol=1e-9)
    assert np.allclose(r.tridiag.subdiag[:m0], want["tsub"][:m0], rtol=1e-9)
    assert np.allclose(r.residual_history[:m0], want["residual_history"][:m0], rtol=1e-9)
    q_gpu = orc.slq(r.tridiag.diag, r.tridiag.subdiag)["value"]
    q_ref = orc.slq(want["tdiag"], want["tsub"])["value"]
    assert q_gpu == pytest.approx(q_ref, rel=1e-6)


def test_mbcg_batched_equals_independent_bitwise(orc):
    n, d = 1000, 3
    x = orc.random_matrix(n, d, 27)
    p = orc.Params(d, 1.0, 0.6, 0.02)
    b = orc.random_matrix(n, 12, 270)
    op = make_op("matern32", x, p, d)
    pc = gk.pivoted_cholesky(op, 20)
    for prec in ("fp64", "fp32", "tf32x3"):
        cfg = gk.CgConfig(200, 1e-6, True, prec, 0)
        batch = gk.batched_pcg(op, b, pc, cfg)
        for c in (0, 5, 11):
            single = gk.batched_pcg(op, b[:, [c]], pc, cfg)[0]
            assert single.iterations_used == batch[c].iterations_used
            assert np.array_equal(single.solution, batch[c].solution)
            assert np.array_equal(single.tridiag.diag, batch[c].tridiag.diag)


def test_mbcg_zero_rhs_and_max_iters(orc):
    n = 200
    x = orc.random_matrix(n, 2, 28)
    p = orc.Params(2, 1.0, 0.5, 0.01)
    op = make_op("rbf", x, p, 2)
    pc = gk.pivoted_cholesky(op, 4)
    b = orc.random_matrix(n, 3, 281)
    b[:, 1] = 0.0
    res = gk.batched_pcg(op, b, pc, gk.CgConfig(3, 1e-12, False, "fp64", 0))
    assert res[1].iterations_used == 0 and res[1].converged and np.linalg.norm(res[1].solution) == 0.0
    assert res[0].iterations_used == 3 and not res[0].converged
    with pytest.raises(gk.InputError):
        gk.batched_pcg(op, b, pc, gk.CgConfig(0, 1e-6))
    with pytest.raises(gk.InputError):
        gk.batched_pcg(op, b, pc, gk.CgConfig(10, 0.0))


def test_preconditioning_does_not_increase_iterations(orc):
    xb = orc.random_matrix(2000, 1, 27)
    x, b = xb[:1000], xb[1000:, 0]
    p = orc.Params(1, 1.0, 0.5, 1e-2)
    op = make_op("rbf", x, p, 1)
    plain = gk.pcg_solve(op, b, gk.IdentityPreconditioner(op), gk.CgConfig(1000, 1e-6, False, "fp64", 0))
    pc = gk.pivoted_cholesky(op, 32)
    pre = gk.pcg_solve(op, b, pc, gk.CgConfig(1000, 1e-6, False, "fp64", 0))
    assert pre.iterations_used <= plain.iterations_used and pre.converged


def test_fp32_refinement_meets_true_residual(orc):
    # solves matching to relative residual 1e-6 (north star), audited in fp64 by the oracle
    n, d = 1500, 3
    x = orc.random_matrix(n, d, 71)
    p = orc.Params(d, 1.0, 0.8, 0.01)
    b = orc.random_matrix(n, 4, 72)
    op = make_op("rbf", x, p, d)
    pc = gk.pivoted_cholesky(op, 30)
    L = pc.factor()
    for prec in ("fp32", "tf32x3"):
        res = gk.batched_pcg(op, b, pc, gk.CgConfig(500, 1e-6, False, prec, 3))
        kx = orc.kernel_apply(orc.RBF, x, p, np.stack([r.solution for r in res], 1))
        for c in range(4):
            assert res[c].converged
            r_true = b[:, c] - kx[:, c]
            num = np.linalg.norm(orc.dplr(0.01, L, r_true)["solve"])
            den = np.linalg.norm(orc.dplr(0.01, L, b[:, c])["solve"])
            assert num / den <= 1.05e-6


# ---------------------------------------------------------------------------
# evaluate_mll (gp_likelihood.hpp:51-103)
# ---------------------------------------------------------------------------
def c1_case():
    w = workloads.config("C1")
    x, y = workloads.generate(w)
    hp = gk.Hyperparameters.from_raw(w.d, w.outputscale, lengthscales=w.lengthscales, noise=w.noise)
    seed = gk.mix_seed(workloads.PROBE_SEED, 1)
    z = gk.make_probes(w.n, w.probes, seed)
    return w, x, y, hp, z


def test_c1_inputs_match_golden():
    g = json.load(open(os.path.join(GOLD, "c1_oracle.json")))
    w, x, y, hp, z = c1_case()
    assert float(np.sum(x * np.arange(1, x.size + 1).reshape(x.shape))) == pytest.approx(g["x_sha"], rel=1e-14)
    assert float(y.sum()) == pytest.approx(g["y_sum"], rel=1e-14)


def _c1_eval(max_iters, precision, backward):
    w, x, y, hp, z = c1_case()
    op = gk.KernelOperator(gk.KernelSpec("rbf"), x, hp)
    pc = gk.pivoted_cholesky_with_derivatives(op, w.rank)
    cfg = gk.MllConfig(gk.CgConfig(max_iters, w.rel_tol, False, precision, 2), True, backward)
    return pc, gk.evaluate_mll(y, op, pc, z, cfg)


def test_c1_reference_faithful_parity():
    """BASELINE C1 exactly as configured (max 100 CG iterations: every solve is truncated before
    reaching tol 1e-6, so the result is the truncated-CG estimate).  The fp64 reference-faithful
    mode reproduces it: identical pivots; mLL and log-det within 1e-6, the gradient within 2e-4.

    The truncated gradient is fixed by fp64 rounding only to ~1e-4 (kappa ~ 4e4, 100
    iterations, no convergence): the oracle's own admissible variants move its outputscale
    component by 1.8e-5 (Dense vs MatrixFree operator, the reference's two modes) and 3.5e-5
    (direct vs expanded distances); GPU variants that differ only in reduction order / libdevice
    exp land at 0.86-1.26e-4 (tools/c1_faithful_err.py).  Converged solves hold the 1e-4 gate
    on every component (test_c1_converged_parity)."""
    g = json.load(open(os.path.join(GOLD, "c1_oracle.json")))
    pc, r = _c1_eval(100, "fp64", "faithful")
    assert pc.pivots() == g["pivots"]
    assert r.value == pytest.approx(g["value"], rel=1e-6)
    assert r.logdet == pytest.approx(g["logdet"], rel=1e-6)
    assert r.solve_iterations == g["solve_iterations"] == 100
    np.testing.assert_allclose(r.gradient, g["gradient"], rtol=2e-4)
    np.testing.assert_allclose(r.forward_gammas, g["forward_gammas"], rtol=1e-4)
    bg = np.array(g["backward_gammas"])
    np.testing.assert_allclose(r.backward_gammas, bg, rtol=1e-3, atol=1e-3 * np.abs(bg).max())


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("backward", ["faithful", "fused"])
def test_c1_truncated_value_and_logdet(precision, backward):
    """Every mode at the truncated C1 configuration: mLL and log-det within 1e-4 (the gradient of
    the fused / fp32 modes is a different estimator of a truncated solve; see the converged test)."""
    g = json.load(open(os.path.join(GOLD, "c1_oracle.json")))
    pc, r = _c1_eval(100, precision, backward)
    assert r.value == pytest.approx(g["value"], rel=1e-4)
    assert r.logdet == pytest.approx(g["logdet"], rel=1e-4)
    assert np.all(np.isfinite(r.gradient))


@pytest.mark.parametrize("precision", ["fp64", "fp32", "tf32x3"])
@pytest.mark.parametrize("backward", ["faithful", "fused"])
def test_c1_converged_parity(precision, backward):
    """C1 with the solves run to tol 1e-6 (max_iters 1000): every precision / backward mode matches
    the oracle within the north-star gate (mLL, log-det, each gradient component 1e-4)."""
    g = json.load(open(os.path.join(GOLD, "c1_converged_oracle.json")))
    pc, r = _c1_eval(1000, precision, backward)
    assert pc.pivots() == g["pivots"]
    assert r.value == pytest.approx(g["value"], rel=1e-4)
    assert r.logdet == pytest.approx(g["logdet"], rel=1e-4)
    np.testing.assert_allclose(r.gradient, g["gradient"], rtol=1e-4)
    if precision != "fp64":
        assert 0.0 <= r.max_true_rel_residual <= 1e-6  # fp64-audited solve residual


@pytest.mark.parametrize("case", range(8))
@pytest.mark.parametrize("backward", ["faithful", "fused"])
def test_grid_evaluate_mll_matches_oracle(orc, case, backward):
    g = json.load(open(os.path.join(GOLD, "grid_oracle.json")))[case]
    x = orc.random_matrix(g["n"], g["d"], g["x_seed"])
    y = np.sin(2 * x[:, 0]) + 0.1 * orc.random_matrix(g["n"], 1, g["y_seed"])[:, 0]
    fam = ["rbf", "matern12", "matern32", "matern52"][g["family"]]
    hp = gk.Hyperparameters.from_raw(g["d"], 1.1, 0.8, 0.05)
    op = gk.KernelOperator(gk.KernelSpec(fam), x, hp)
    pc = gk.pivoted_cholesky_with_derivatives(op, g["rank"])
    z = gk.make_probes(g["n"], g["l"], g["probe_seed"])
    r = gk.evaluate_mll(y, op, pc, z, gk.MllConfig(gk.CgConfig(200, 1e-8, False, "fp64", 0), True, backward))
    # solves to rel_tol 1e-8: the value is determined to ~1e-9 (kernel entries differ from the
    # oracle's by the DMMA Gram rounding, ~1e-16 relative), so the gate is the solve tolerance
    assert r.value == pytest.approx(g["value"], rel=1e-8)
    np.testing.assert_allclose(r.gradient, g["gradient"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(r.forward_gammas, g["forward_gammas"], rtol=1e-7, atol=1e-12)


@pytest.mark.parametrize("precision", ["fp64", "tf32x3"])
def test_wide_faithful_backward_matches_oracle(orc, precision):
    """Reference-faithful backward with (d+1) l = 96 right-hand sides: the fused single-rank CG
    iteration runs its Woodbury G1s / G2s in two column groups (64 + 32) and the beta/p update
    over all 96 columns; value, log-det and every gradient component match the oracle."""
    n, d, l = 640, 3, 24
    x = orc.random_matrix(n, d, 3100)
    y = np.cos(3 * x[:, 1]) + 0.1 * orc.random_matrix(n, 1, 3101)[:, 0]
    p = orc.Params(d, 1.0, 0.6, 0.03)
    z = orc.make_probes(n, l, 3102)
    want = orc.evaluate_mll(orc.MATERN52, x, p, y, z, seed=3102, prec="pivchol", rank=12, max_iters=400,
                            rel_tol=1e-9)
    op = make_op("matern52", x, p, d)
    pc = gk.pivoted_cholesky_with_derivatives(op, 12)
    r = gk.evaluate_mll(y, op, pc, gk.make_probes(n, l, 3102),
                        gk.MllConfig(gk.CgConfig(400, 1e-9, False, precision, 2), True, "faithful"))
    tol = 1e-8 if precision == "fp64" else 1e-5
    assert r.value == pytest.approx(want["value"], rel=tol)
    assert r.logdet == pytest.approx(want["logdet"], rel=tol)
    np.testing.assert_allclose(r.gradient, want["gradient"], rtol=100 * tol, atol=1e-8)


def test_identity_and_unshared_probes_match_oracle(orc):
    n, d = 250, 2
    x = orc.random_matrix(n, d, 85)
    y = orc.random_matrix(n, 1, 86)[:, 0]
    p = orc.Params(d, 1.0, 0.7, 0.05)
    z = orc.make_probes(n, 4, 9)
    for share in (True, False):
        want = orc.evaluate_mll(orc.RBF, x, p, y, z, seed=9, prec="identity", share_probes=share, max_iters=300,
                                rel_tol=1e-9)
        op = make_op("rbf", x, p, d)
        ip = gk.IdentityPreconditioner(op)
        for backward in ("faithful", "fused"):
            r = gk.evaluate_mll(y, op, ip, gk.ProbeBatch(z, 9, 4),
                                gk.MllConfig(gk.CgConfig(300, 1e-9, False, "fp64", 0), share, backward))
            assert r.value == pytest.approx(want["value"], rel=1e-9)
            np.testing.assert_allclose(r.gradient, want["gradient"], rtol=1e-6, atol=1e-9)


def test_line_search_frozen_preconditioner(orc):
    # preconditioner from the step's start theta, K_hat at a trial theta (optimizer.hpp:437 vs :450-451)
    n, d = 300, 2
    x = orc.random_matrix(n, d, 87)
    y = orc.random_matrix(n, 1, 88)[:, 0]
    p0 = gk.Hyperparameters.from_raw(d, 1.0, 0.7, 0.05)
    p1 = gk.Hyperparameters.from_raw(d, 1.2, 0.6, 0.04)
    op = gk.KernelOperator(gk.KernelSpec("matern52"), x, p0)
    pc = gk.pivoted_cholesky_with_derivatives(op, 10)
    op.with_params(p1)
    z = gk.make_probes(n, 6, 3)
    cfg = gk.MllConfig(gk.CgConfig(300, 1e-10, False, "fp64", 0), True, "faithful")
    r = gk.evaluate_mll(y, op, pc, z, cfg)
    v, gr = orc.mll_exact(orc.MATERN52, x, orc.Params(d, 1.2, 0.6, 0.04), y)
    assert r.value == pytest.approx(v, rel=5e-2)
    assert np.all(np.isfinite(r.gradient))


def test_evaluate_rejects_bad_input(orc):
    n = 64
    x = orc.random_matrix(n, 1, 89)
    op = make_op("rbf", x, orc.Params(1), 1)
    pc = gk.pivoted_cholesky_with_derivatives(op, 4)
    z = gk.make_probes(n, 2, 1)
    bad = np.zeros(n)
    bad[0] = np.inf
    with pytest.raises(gk.InputError):
        gk.evaluate_mll(bad, op, pc, z, gk.MllConfig())
    with pytest.raises(gk.InputError):
        gk.evaluate_mll(np.zeros(n + 1), op, pc, z, gk.MllConfig())


@pytest.mark.parametrize("precision", ["fp64", "tf32x3"])
def test_c1_auto_backward_follows_convergence(precision):
    """The default backward mode ('auto') uses the fused bilinear pass only when every forward
    solve converged: z' K^-1 dK z = s' dK z needs s = K^-1 z.  At BASELINE C1 as configured
    every solve is truncated at 100 iterations, and the fused estimator built on the truncated
    probe solves is ~3x further from the converged gradient than the reference's own truncated
    estimator (profiles/r2_c1_fused_truncation.txt); 'auto' then reproduces the reference-faithful
    per-RHS solves, bitwise the faithful mode, within the C1 gate of the faithful test."""
    g = json.load(open(os.path.join(GOLD, "c1_oracle.json")))
    _, auto = _c1_eval(100, precision, "auto")
    _, faith = _c1_eval(100, precision, "faithful")
    assert auto.unconverged_columns > 0 and auto.backward_mode_used == "faithful"
    assert np.array_equal(auto.gradient, faith.gradient) and auto.value == faith.value
    assert auto.value == pytest.approx(g["value"], rel=1e-4)
    if precision == "fp64":
        np.testing.assert_allclose(auto.gradient, g["gradient"], rtol=2e-4)
    else:
        # a reduced-precision operator perturbs the truncated Krylov iterates themselves (kappa ~ 4e4,
        # nothing converged): the truncated gradient then moves by the order of the truncation error --
        # measured 1.1-3.3x of it with the round-1 accumulation order, 1.0-4.6x with round 2's fp32
        # second-level sums; at most 1.7e-3 relative (the small outputscale component) in either case
        ref = np.array(g["gradient"])
        trunc = np.abs(ref - np.array(json.load(open(os.path.join(GOLD, "c1_converged_oracle.json")))["gradient"]))
        assert np.all(np.abs(auto.gradient - ref) <= 8.0 * trunc + 1e-4 * np.abs(ref))
        np.testing.assert_allclose(auto.gradient, ref, rtol=3e-3)
    # converged solves: 'auto' is the fused pass
    _, conv = _c1_eval(1000, precision, "auto")
    assert conv.unconverged_columns == 0 and conv.backward_mode_used == "fused"


def test_fused_split_reduction_is_bitwise_the_separate_launch(orc, monkeypatch):
    """The CG loop's p'Ap kernel sums the fused MVM's split-K partials itself (same split order
    from 0.0 as reduce_splits): every iterate, hence the whole evaluation, is bitwise the one with
    the separate reduction launch (GPK_FUSE_REDUCE=0)."""
    n, d, l = 3000, 9, 6
    x = orc.random_matrix(n, d, 91)
    y = np.sin(x[:, 0]) + 0.1 * orc.random_matrix(n, 1, 92)[:, 0]
    hp = gk.Hyperparameters.from_raw(d, 1.0, 1.5, 0.05)
    z = gk.make_probes(n, l, gk.mix_seed(3, 1))
    cfg = gk.MllConfig(gk.CgConfig(200, 1e-6, False, "tf32x3", 2), True, "fused")
    got = []
    for flag in ("1", "0"):
        monkeypatch.setenv("GPK_FUSE_REDUCE", flag)
        op = gk.KernelOperator(gk.KernelSpec("matern32"), x, hp)  # the switch is read per context
        pc = gk.pivoted_cholesky_with_derivatives(op, 20)
        got.append(gk.evaluate_mll(y, op, pc, z, cfg))
    a, b = got
    assert a.value == b.value and a.logdet == b.logdet
    assert np.array_equal(a.gradient, b.gradient)
    assert np.array_equal(a.forward_cg_iterations, b.forward_cg_iterations)
    assert b.gpu_launches - a.gpu_launches >= a.solve_iterations  # one launch less per iteration
