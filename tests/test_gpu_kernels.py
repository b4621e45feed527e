"""GPU parity of the kernel operator, pivoted Cholesky, Woodbury and derivative
factors against the CPU oracle (same seeded inputs), through the C-ABI."""
import math

import numpy as np
import pytest

import paper_2107_00243_b200 as gk

pytestmark = pytest.mark.gpu

FAMS = ["rbf", "matern12", "matern32", "matern52"]


def op_for(orc, fam, x, p, precision="fp64"):
    hp = gk.Hyperparameters(p.log_o, np.array(p.log_ls), p.log_noise)
    return gk.KernelOperator(gk.KernelSpec(fam), x, hp, precision=precision)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("fam", FAMS)
@pytest.mark.parametrize("n,d,t", [(1, 1, 1), (100, 2, 3), (1000, 3, 9), (2051, 9, 51), (700, 18, 65), (300, 32, 130)])
def test_mvm_fp64_matches_oracle(orc, fam, n, d, t):
    x = orc.random_matrix(n, d, 100 + n + d)
    p = orc.Params(d, 1.3, 0.9 * math.sqrt(d), 0.05)
    v = orc.random_matrix(n, t, 7 + t)
    want = orc.kernel_apply(orc.FAMILIES[fam], x, p, v)
    op = op_for(orc, fam, x, p)
    got = op.apply(v, precision="fp64")
    assert rel(got, want) < 1e-12


@pytest.mark.parametrize("fam", FAMS)
@pytest.mark.parametrize("n,d,t", [(1000, 3, 9), (2051, 9, 51), (700, 18, 65), (300, 32, 130), (129, 1, 1)])
@pytest.mark.parametrize("precision", ["fp32", "tf32x3"])
def test_mvm_fp32_matches_oracle(orc, fam, n, d, t, precision):
    # fp32 entries (direct differences, SFU exp); contraction on CUDA cores (fp32) or on the
    # tcgen05 tensor cores in 3xTF32 split precision (tf32x3); fp64 across accumulation groups
    x = orc.random_matrix(n, d, 200 + n)
    p = orc.Params(d, 1.0, 0.8 * math.sqrt(d), 0.01)
    v = orc.random_matrix(n, t, 9)
    want = orc.kernel_apply(orc.FAMILIES[fam], x, p, v)
    got = op_for(orc, fam, x, p).apply(v, precision=precision)
    assert rel(got, want) < (2e-6 if precision == "fp32" else 3e-6)
    # per column too
    for c in range(t):
        assert rel(got[:, c], want[:, c]) < (5e-6 if precision == "fp32" else 1e-5)


@pytest.mark.parametrize("fam", ["rbf", "matern32", "matern52"])
@pytest.mark.parametrize("n,d,t", [(1000, 3, 9), (2051, 9, 51), (700, 18, 65), (300, 32, 130), (129, 1, 1),
                                   (4100, 11, 8), (640, 30, 51), (5000, 18, 51)])
@pytest.mark.parametrize("variant", ["direct", "gram"])
def test_mvm_tc_variants_match_oracle(orc, fam, n, d, t, variant):
    # both kernel-entry strategies of the tensor-core MVM: fp32 direct differences, and
    # the expanded form with the cross term on the tensor cores (gpk_mvm_tcg.cuh)
    x = orc.random_matrix(n, d, 300 + n)
    p = orc.Params(d, 1.0, 0.8 * math.sqrt(d), 0.01)
    v = orc.random_matrix(n, t, 11)
    want = orc.kernel_apply(orc.FAMILIES[fam], x, p, v)
    op = op_for(orc, fam, x, p).set_mvm_variant(variant)
    got = op.apply(v, precision="tf32x3")
    # the Gram MMA runs on d + 2 augmented coordinates (<= 32): d > 30 falls back to direct
    assert op.mvm_variant()[0] == (variant if d <= 30 else "direct")
    assert rel(got, want) < 3e-6
    for c in range(t):
        assert rel(got[:, c], want[:, c]) < 1e-5


def test_mvm_variant_auto_selection(orc):
    # auto: Gram for moderate coordinate norms, direct differences for large ones and Matern-1/2
    x = orc.random_matrix(2000, 18, 41)
    small = op_for(orc, "matern32", x, orc.Params(18, 1.0, 2.0, 0.01))
    assert small.mvm_variant()[0] == "gram"
    big = op_for(orc, "matern32", 100.0 * x, orc.Params(18, 1.0, 2.0, 0.01))
    assert big.mvm_variant()[0] == "direct"
    m12 = op_for(orc, "matern12", x, orc.Params(18, 1.0, 2.0, 0.01)).set_mvm_variant("gram")
    assert m12.mvm_variant()[0] == "direct"
    # clustered near-duplicate points (C4-like): Gram stays accurate near s = 0 where forced
    xc = np.repeat(orc.random_matrix(64, 3, 42), 20, axis=0) + 1e-3 * orc.random_matrix(1280, 3, 43)
    p = orc.Params(3, 1.0, 0.3, 0.01)
    v = orc.random_matrix(1280, 5, 44)
    want = orc.kernel_apply(orc.FAMILIES["matern52"], xc, p, v)
    op = op_for(orc, "matern52", xc, p).set_mvm_variant("gram")
    assert rel(op.apply(v, precision="tf32x3"), want) < 3e-6


@pytest.mark.parametrize("fam", FAMS)
@pytest.mark.parametrize("precision,tol", [("fp64", 1e-11), ("fp32", 5e-6)])
def test_deriv_mvm_matches_oracle(orc, fam, precision, tol):
    n, d = 600, 3
    x = orc.random_matrix(n, d, 31)
    p = orc.Params(d, 1.4, 0.8, 0.05)
    v = orc.random_matrix(n, 5, 32)
    op = op_for(orc, fam, x, p)
    for which in range(d + 2):
        want = orc.kernel_apply(orc.FAMILIES[fam], x, p, v, which=which)
        got = op.deriv_apply(which, v, precision=precision)
        assert rel(got, want) < tol, (which, rel(got, want))


def test_mvm_columns_are_independent_bitwise(orc):
    # a column's result never depends on the other columns of the block (batched_pcg contract)
    x = orc.random_matrix(1500, 11, 5)
    p = orc.Params(11, 1.0, 2.0, 0.01)
    v = orc.random_matrix(1500, 65, 6)
    op = op_for(orc, "matern32", x, p)
    for prec in ("fp32", "fp64", "tf32x3"):
        full = op.apply(v, precision=prec)
        for cols in ([0], [3, 17], list(range(40, 51))):
            part = op.apply(v[:, cols], precision=prec)
            assert np.array_equal(part, full[:, cols])


def test_mvm_rejects_bad_input(orc):
    x = orc.random_matrix(8, 1, 7)
    op = op_for(orc, "rbf", x, orc.Params(1))
    with pytest.raises(gk.InputError):
        op.apply(np.zeros(9))
    bad = np.zeros(8)
    bad[3] = np.nan
    with pytest.raises(gk.InputError, match="non-finite"):
        op.apply(bad)
    with pytest.raises(gk.InputError):
        op.deriv_apply(5, np.zeros(8))


@pytest.mark.parametrize("fam", FAMS)
def test_kernel_columns_match_oracle(orc, fam):
    n, d = 513, 3
    x = orc.random_matrix(n, d, 41)
    p = orc.Params(d, 1.2, 0.7, 0.05)
    op = op_for(orc, fam, x, p)
    f = orc.FAMILIES[fam]
    for i in (0, 7, n - 1):
        assert rel(op.kernel_column(i), orc.kernel_column(f, x, p, i)) < 1e-15
        for w in range(d + 2):
            want = orc.kernel_column(f, x, p, i, which=w)
            got = op.kernel_deriv_column(w, i)
            assert np.allclose(got, want, rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("fam,n,d,rank", [("rbf", 2048, 3, 16), ("matern32", 1000, 2, 64), ("matern52", 777, 5, 40),
                                          ("matern12", 300, 1, 30)])
def test_pivoted_cholesky_pivots_identical(orc, fam, n, d, rank):
    x = orc.random_matrix(n, d, 50 + rank)
    p = orc.Params(d, 1.1, 0.6, 0.01)
    want = orc.pivoted_cholesky(rank, family=orc.FAMILIES[fam], x=x, p=p)
    op = op_for(orc, fam, x, p)
    pc, rem = gk.pivoted_cholesky(op, rank, want_remaining=True)
    assert pc.pivots() == list(want["pivots"])
    assert pc.rank() == want["rank"]
    assert rel(pc.factor(), want["L"]) < 1e-12
    assert np.allclose(rem, want["remaining"], rtol=1e-10, atol=1e-13)


def test_pivoted_cholesky_diag_tol_and_errors(orc):
    x = (np.arange(50) / 49.0)[:, None]
    p = orc.Params(1, 1.0, 0.5, 0.01)
    op = op_for(orc, "rbf", x, p)
    want = orc.pivoted_cholesky(50, diag_tol=1e-6, family=orc.RBF, x=x, p=p)
    pc = gk.pivoted_cholesky(op, 50, diag_tol=1e-6)
    assert pc.rank() == want["rank"] < 50
    assert pc.pivots() == list(want["pivots"])
    with pytest.raises(gk.InputError):
        gk.pivoted_cholesky(op, 51)
    with pytest.raises(gk.InputError):
        gk.pivoted_cholesky(op, 3, noise_variance=0.0)


@pytest.mark.parametrize("fam", ["rbf", "matern32"])
def test_deriv_factors_and_traces_match_oracle(orc, fam):
    n, d, rank = 400, 2, 12
    x = orc.random_matrix(n, d, 42)
    p = orc.Params(d, 1.2, 0.7, 0.05)
    op = op_for(orc, fam, x, p)
    pc = gk.pivoted_cholesky_with_derivatives(op, rank)
    ref = orc.pivoted_cholesky(rank, family=orc.FAMILIES[fam], x=x, p=p)
    dls = orc.deriv_factors(orc.FAMILIES[fam], x, p, ref["L"], ref["pivots"])
    L = ref["L"]
    for w in range(d + 1):
        assert rel(pc.deriv_factor(w), dls[w]) < 1e-11
        want = orc.dplr_trace_inv_deriv(0.05, L, dls[w])
        assert pc.trace_inv_deriv(w) == pytest.approx(want, rel=1e-10, abs=1e-12)
    # noise: tr(P^-1)
    assert pc.trace_inv_deriv(d + 1) == pytest.approx(orc.dplr(0.05, L, np.ones(n))["trace_inv"], rel=1e-12)


def test_woodbury_solve_and_logdet(orc):
    n, d, rank = 900, 3, 25
    x = orc.random_matrix(n, d, 43)
    p = orc.Params(d, 1.0, 0.5, 0.02)
    op = op_for(orc, "rbf", x, p)
    pc = gk.pivoted_cholesky(op, rank)
    L = pc.factor()
    v = orc.random_matrix(n, 4, 44)
    for c in range(4):
        want = orc.dplr(0.02, L, v[:, c])
        assert rel(pc.solve(v[:, c]), want["solve"]) < 1e-12
    assert pc.logdet() == pytest.approx(orc.dplr(0.02, L, v[:, 0])["logdet"], rel=1e-12)
    # rank 0: P = sigma^2 I
    p0 = gk.pivoted_cholesky(op, 0)
    assert np.allclose(p0.solve(v[:, 0]), v[:, 0] / 0.02, rtol=1e-15)
    assert p0.logdet() == pytest.approx(n * math.log(0.02), rel=1e-14)


@pytest.mark.parametrize("variant,fam,d", [("gram", "matern32", 18), ("gram", "rbf", 9), ("direct", "matern52", 3)])
def test_tcg_persistent_multi_unit_ctas_bitwise(orc, monkeypatch, variant, fam, d):
    """The persistent tcgen05 MVM grid runs contiguous (row block, split) units per CTA.  Capping
    the grid (test hook GPK_TCG_CTAS) forces many units per CTA -- row-block changes (the CTA
    barrier, the new TMEM row operand) and same-row split changes (flipped mbarrier phases, the
    unit-indexed split slots, the accumulator reset) -- and must give bitwise the full grid's
    rows, which match the oracle (these paths only ran at the C2 bench shape)."""
    n, t = 9000, 51  # 71 row blocks x several 64-tile splits
    x = orc.random_matrix(n, d, 77)
    p = orc.Params(d, 1.0, 0.9 * math.sqrt(d), 0.01)
    v = orc.random_matrix(n, t, 78)
    full = op_for(orc, fam, x, p).set_mvm_variant(variant)
    want_gpu = full.apply(v, precision="tf32x3")
    assert full.mvm_variant()[0] == variant
    for cap in (7, 29):
        monkeypatch.setenv("GPK_TCG_CTAS", str(cap))
        capped = op_for(orc, fam, x, p).set_mvm_variant(variant)
        got = capped.apply(v, precision="tf32x3")
        assert np.array_equal(got, want_gpu), cap
    # strided unit order (what large n uses so that all CTAs share a j-range in the L2): the same
    # (row block, split) units with the same split slots, handed out b, b + G, b + 2 G, ... -- every
    # unit then starts a new row block -- bitwise the contiguous order
    for cap in (7, 29, 0):
        if cap:
            monkeypatch.setenv("GPK_TCG_CTAS", str(cap))
        else:
            monkeypatch.delenv("GPK_TCG_CTAS")
        monkeypatch.setenv("GPK_TCG_ORDER", "1")
        strided = op_for(orc, fam, x, p).set_mvm_variant(variant)
        got = strided.apply(v, precision="tf32x3")
        assert np.array_equal(got, want_gpu), ("strided", cap)
    monkeypatch.delenv("GPK_TCG_ORDER")
    rows = np.arange(0, n, 37)
    want = orc.kernel_apply_rows(orc.FAMILIES[fam], x, p, rows, v)
    assert rel(want_gpu[rows], want) < 3e-6


@pytest.mark.gpu
@pytest.mark.parametrize("n,count,seed", [(1, 1, 0), (311, 1, 5489), (312, 2, 1), (313, 3, 17), (1000, 7, 2 ** 63 + 11),
                                           (16384, 50, 0x9E3779B97F4A7C15)])
def test_device_probes_equal_host_stream(orc, n, count, seed):
    """gpk_make_probes_device (block-parallel MT19937-64 on the device, gpk_probes.cu) is bitwise
    the host std::mt19937_64 stream of trace_estimation.hpp:27-36 -- and the oracle's own."""
    x = orc.random_matrix(max(n, 2), 2, 1)[:n]
    op = gk.KernelOperator(gk.KernelSpec("rbf"), x, gk.Hyperparameters.from_raw(2, 1.0, 1.0, 0.1))
    z = gk.make_probes_device(op, count, seed).cpu().numpy()  # (count, n)
    host = gk.make_probes(n, count, seed).probes
    assert z.shape == (count, n)
    assert np.array_equal(z.T, host)
    assert np.array_equal(host, orc.make_probes(n, count, seed))
