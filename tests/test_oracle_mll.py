"""Pins the oracle's composite evaluate_mll.  The reference has no test for it
(test_gp_likelihood.cpp is an empty stub), so the SPEC's unimplemented
acceptance items are the known answers: n=1 closed forms,
deterministic collapse with P = K_hat (acceptance #2), agreement with the dense
oracle and gradient vs finite differences of the dense mLL (#8)."""
import math

import numpy as np
import pytest


def test_n1_closed_form(orc):
    o, s2, yv = 1.3, 0.2, 0.7
    p = orc.Params(1, o, 1.0, s2)
    x = np.array([[0.4]])
    z = orc.make_probes(1, 1, 5)
    r = orc.evaluate_mll(orc.RBF, x, p, np.array([yv]), z, prec="pivchol", rank=0, max_iters=10)
    k = o * o + s2
    assert r["value"] == pytest.approx(-0.5 * (yv * yv / k + math.log(k) + math.log(2 * math.pi)), rel=1e-13)
    g = 0.5 * (yv * yv / k ** 2 - 1.0 / k)
    assert r["gradient"][0] == pytest.approx(g * 2 * o * o, rel=1e-12)
    assert r["gradient"][1] == pytest.approx(0.0, abs=1e-14)
    assert r["gradient"][2] == pytest.approx(g * s2, rel=1e-12)


@pytest.mark.parametrize("fam", [0, 2, 3])
def test_deterministic_collapse(orc, fam):
    # SPEC acceptance #2: P = K_hat, m = n, n = 64 -> dense oracle to rel 1e-8
    x = orc.random_matrix(64, 2, 77)
    y = orc.random_matrix(64, 1, 78)[:, 0]
    p = orc.Params(2, 1.1, 0.8, 0.05)
    z = orc.make_probes(64, 4, orc.mix_seed(17, 1))
    r = orc.evaluate_mll(fam, x, p, y, z, prec="exact", max_iters=64, rel_tol=1e-12, mode=orc.DENSE)
    v, g = orc.mll_exact(fam, x, p, y)
    assert r["value"] == pytest.approx(v, rel=1e-8)
    np.testing.assert_allclose(r["gradient"], g, rtol=1e-8, atol=1e-10)


def test_dense_and_matrix_free_agree(orc):
    x = orc.random_matrix(96, 3, 79)
    y = orc.random_matrix(96, 1, 80)[:, 0]
    p = orc.Params(3, 1.0, 0.6, 0.02)
    z = orc.make_probes(96, 6, 3)
    a = orc.evaluate_mll(orc.MATERN32, x, p, y, z, rank=8, mode=orc.DENSE)
    b = orc.evaluate_mll(orc.MATERN32, x, p, y, z, rank=8, mode=orc.MATRIX_FREE)
    assert a["value"] == pytest.approx(b["value"], rel=1e-10)
    np.testing.assert_allclose(a["gradient"], b["gradient"], rtol=1e-7, atol=1e-9)
    # rounding differs between the two storage modes; iteration counts may differ by one at the threshold
    assert np.max(np.abs(a["forward_cg_iterations"] - b["forward_cg_iterations"])) <= 1


def test_matches_dense_oracle_1d_rbf(orc):
    # n=500 1-d RBF, rank-64 pivoted Cholesky, m=200 -> rel 1e-3 of the dense oracle
    n = 500
    x = np.sort(orc.random_matrix(n, 1, 81), axis=0)
    y = np.sin(3 * x[:, 0]) + 0.1 * orc.random_matrix(n, 1, 82)[:, 0]
    p = orc.Params(1, 1.0, 0.5, 0.01)
    z = orc.make_probes(n, 64, orc.mix_seed(17, 1))
    r = orc.evaluate_mll(orc.RBF, x, p, y, z, rank=64, max_iters=200)
    v, _ = orc.mll_exact(orc.RBF, x, p, y)
    assert r["value"] == pytest.approx(v, rel=1e-3)


def test_gradient_vs_dense_fd(orc):
    # SPEC acceptance #8: n=256, 128 probes, rank-128 preconditioner, each component within
    # rel 5e-2 of central FD of the dense mLL (step 1e-4 in log space)
    n = 256
    x = orc.random_matrix(n, 2, 83)
    y = np.sin(x[:, 0]) * np.cos(x[:, 1]) + 0.1 * orc.random_matrix(n, 1, 84)[:, 0]
    p = orc.Params(2, 1.2, 0.9, 0.05)
    z = orc.make_probes(n, 128, orc.mix_seed(17, 1))
    r = orc.evaluate_mll(orc.RBF, x, p, y, z, rank=128, max_iters=200)
    h = 1e-4
    for w in range(4):
        def f(delta):
            q = orc.Params(2, 1.2, 0.9, 0.05)
            if w == 0:
                q.log_o += delta
            elif w <= 2:
                q.log_ls = q.log_ls.copy()
                q.log_ls[w - 1] += delta
            else:
                q.log_noise += delta
            return orc.mll_exact(orc.RBF, x, q, y)[0]
        fd = (f(h) - f(-h)) / (2 * h)
        assert r["gradient"][w] == pytest.approx(fd, rel=5e-2)


def test_unshared_probes_and_identity(orc):
    x = orc.random_matrix(64, 2, 85)
    y = orc.random_matrix(64, 1, 86)[:, 0]
    p = orc.Params(2, 1.0, 0.7, 0.05)
    z = orc.make_probes(64, 4, 9)
    a = orc.evaluate_mll(orc.RBF, x, p, y, z, seed=9, prec="identity", share_probes=False)
    b = orc.evaluate_mll(orc.RBF, x, p, y, z, seed=9, prec="identity", share_probes=True)
    assert a["value"] == b["value"]  # the forward pass is identical
    assert np.all(np.isfinite(a["gradient"])) and not np.array_equal(a["gradient"], b["gradient"])
