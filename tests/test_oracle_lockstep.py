"""The oracle's lock-step batched evaluation (used to make the BASELINE-size C2 fixtures,
tests/golden/make_golden_big.py) is bitwise the oracle's per-column reference restatement.

batched_pcg's contract (krylov.hpp:131-153) is that every column is bitwise pcg_solve; the
lock-step driver advances all columns of a phase together and applies the operator to the
block (KernelOperator::apply_block, a cache-blocked GEMM over the stored MatrixFree kernel
block with each output's sequential sum kept).  So the C2 goldens carry the same numbers the
per-column MatrixFree restatement of gp_likelihood.hpp:51-103 would produce, only faster."""
import numpy as np
import pytest

KEYS = ("value", "logdet", "quad", "gradient", "forward_gammas", "backward_gammas", "forward_cg_iterations", "u",
        "total_cg_iterations", "solve_iterations", "value_sample_variance")


@pytest.mark.parametrize("fam", [0, 1, 2, 3])
@pytest.mark.parametrize("rank", [0, 9])
@pytest.mark.parametrize("share", [True, False])
def test_lockstep_evaluate_bitwise_equals_per_column(orc, fam, rank, share):
    n, d, l = 301, 3, 5  # 301: a partial 16-row register tile and two 256-row GEMM blocks
    x = orc.random_matrix(n, d, 40 + fam)
    y = np.sin(2 * x[:, 0]) + 0.1 * orc.random_matrix(n, 1, 41)[:, 0]
    p = orc.Params(d, 1.1, 0.8, 0.05)
    z = orc.make_probes(n, l, 9)
    a = orc.evaluate_mll(fam, x, p, y, z, seed=9, prec="pivchol", rank=rank, mode=orc.MATRIX_FREE, max_iters=400,
                         rel_tol=1e-8, share_probes=share)
    b = orc.evaluate_mll(fam, x, p, y, z, seed=9, prec="pivchol", rank=rank, mode=orc.CACHED, max_iters=400,
                         rel_tol=1e-8, share_probes=share, lockstep=True)
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), k
    assert a["total_cg_iterations"] < 400 * (l + 1 + (d + 2) * l)  # converged, not capped


def test_lockstep_truncated_and_identity(orc):
    # every column hits max_iters (the BASELINE C1 regime) and the identity preconditioner
    n, d, l = 200, 2, 4
    x = orc.random_matrix(n, d, 50)
    y = orc.random_matrix(n, 1, 51)[:, 0]
    p = orc.Params(d, 1.0, 0.3, 1e-3)
    z = orc.make_probes(n, l, 3)
    for prec in ("identity", "pivchol"):
        a = orc.evaluate_mll(0, x, p, y, z, seed=3, prec=prec, rank=4, max_iters=7)
        b = orc.evaluate_mll(0, x, p, y, z, seed=3, prec=prec, rank=4, mode=orc.CACHED, max_iters=7, lockstep=True)
        for k in KEYS:
            assert np.array_equal(a[k], b[k]), (prec, k)
        assert a["solve_iterations"] == 7


def test_block_apply_and_row_subset_bitwise(orc):
    n, d, t = 517, 5, 13
    x = orc.random_matrix(n, d, 60)
    p = orc.Params(d, 1.2, 1.1, 0.02)
    v = orc.random_matrix(n, t, 61)
    for fam in (0, 1, 2, 3):
        want = orc.kernel_apply(fam, x, p, v)
        assert np.array_equal(orc.kernel_apply_block(fam, x, p, v, mode=orc.CACHED), want)
        rows = np.array([0, 1, 127, 128, 255, 256, 400, n - 1])
        assert np.array_equal(orc.kernel_apply_rows(fam, x, p, rows, v), want[rows])


def test_lockstep_rejects_bad_input(orc):
    # the operator's input check (kernels.hpp:285-288) fires on the block apply as on apply()
    n = 64
    x = orc.random_matrix(n, 1, 70)
    y = np.ones(n)
    y[5] = np.inf
    for mode, lockstep in ((orc.MATRIX_FREE, False), (orc.CACHED, True)):
        with pytest.raises(orc.InputError, match="non-finite"):
            orc.evaluate_mll(0, x, orc.Params(1, 1.0, 0.5, 0.01), y, orc.make_probes(n, 2, 1), prec="identity",
                             mode=mode, lockstep=lockstep)
