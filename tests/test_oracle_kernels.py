"""Pins the CPU oracle's kernel operator to the reference's own known-answer
tests (proj/tests/test_kernels.cpp).  Test infrastructure: checks the checker."""
import math

import numpy as np
import pytest

ALL = ["rbf", "matern12", "matern32", "matern52", "ratquad"]


def test_closed_forms(orc):
    # test_kernels.cpp:17-34 (kernel_value via two-point kernel columns)
    p = orc.Params(1)
    col = lambda fam, a, b: orc.kernel_column(orc.FAMILIES[fam], np.array([[a], [b]]), p, 0)[1]
    assert col("rbf", 0.3, 0.3) == pytest.approx(1.0)
    assert col("rbf", 0.0, math.sqrt(2 * math.log(2))) == pytest.approx(0.5, rel=1e-12)
    assert col("matern12", 0.0, 1.0) == pytest.approx(math.exp(-1.0), rel=1e-12)
    assert col("matern32", 0.5, 0.5) == pytest.approx(1.0)
    assert col("ratquad", 0.0, 1.0) == pytest.approx(1.0 / 1.5, rel=1e-12)


def test_stationarity_bound(orc):
    # test_kernels.cpp:36-47
    x = orc.random_matrix(2, 3, 3)
    p = orc.Params(3, 1.7, 0.8)
    for fam in ALL:
        c = orc.kernel_column(orc.FAMILIES[fam], x, p, 0)
        assert c[0] == pytest.approx(1.7 ** 2)
        assert c[1] <= 1.7 ** 2 + 1e-15


@pytest.mark.parametrize("fam", ["rbf", "matern32"])
def test_matrix_free_matches_dense(orc, fam):
    # test_kernels.cpp:55-68 — uneven 7-row blocks, 1e-12
    x = orc.random_matrix(64, 2, 5)
    p = orc.Params(2, 1.3, 0.9, 0.05)
    v = np.random.default_rng(5).standard_normal(64)
    dense = orc.dense(orc.FAMILIES[fam], x, p)
    want = dense @ v
    got_dense = orc.kernel_apply(orc.FAMILIES[fam], x, p, v, mode=orc.DENSE)[:, 0]
    got_free = orc.kernel_apply(orc.FAMILIES[fam], x, p, v, mode=orc.MATRIX_FREE, block_rows=7)[:, 0]
    assert np.linalg.norm(got_dense - want) / np.linalg.norm(want) < 1e-12
    assert np.linalg.norm(got_free - want) / np.linalg.norm(want) < 1e-12


def test_trivial_cases(orc):
    # test_kernels.cpp:70-81
    p = orc.Params(1, 1.5, 1.0, 0.3)
    out = orc.kernel_apply(orc.RBF, np.array([[0.4]]), p, np.ones(1), mode=orc.DENSE)
    assert out[0, 0] == pytest.approx(1.5 ** 2 + 0.3, rel=1e-14)
    x = orc.random_matrix(64, 2, 6)
    assert np.linalg.norm(orc.kernel_apply(orc.RBF, x, orc.Params(2), np.zeros(64))) == 0.0


def test_rejects_bad_input(orc):
    # test_kernels.cpp:83-91
    x = orc.random_matrix(8, 1, 7)
    p = orc.Params(1)
    bad = np.zeros(8)
    bad[3] = np.nan
    with pytest.raises(orc.InputError):
        orc.kernel_apply(orc.RBF, x, p, bad)
    with pytest.raises(orc.InputError):
        orc.kernel_apply(orc.RBF, x, p, np.zeros(8), which=5)


def test_symmetry(orc):
    # test_kernels.cpp:93-101
    x = orc.random_matrix(48, 3, 8)
    p = orc.Params(3, 1.1, 0.7, 0.02)
    rng = np.random.default_rng(8)
    for _ in range(5):
        u, v = rng.standard_normal(48), rng.standard_normal(48)
        au = orc.kernel_apply(orc.MATERN52, x, p, u)[:, 0]
        av = orc.kernel_apply(orc.MATERN52, x, p, v)[:, 0]
        assert u @ av == pytest.approx(v @ au, rel=1e-11)


@pytest.mark.parametrize("fam", ALL)
def test_dense_psd(orc, fam):
    # test_kernels.cpp:103-113
    x = orc.random_matrix(96, 2, 9)
    p = orc.Params(2, 1.0, 0.6, 1e-300)
    ev = np.linalg.eigvalsh(orc.dense(orc.FAMILIES[fam], x, p))
    assert ev.min() > -1e-10 * ev.max()


def test_noise_derivative_identity(orc):
    # test_kernels.cpp:115-120
    x = orc.random_matrix(16, 2, 10)
    v = np.random.default_rng(10).standard_normal(16)
    out = orc.kernel_apply(orc.RBF, x, orc.Params(2), v, which=3)[:, 0]
    assert np.linalg.norm(out - v) == 0.0


@pytest.mark.parametrize("fam", ALL)
@pytest.mark.parametrize("which", [0, 1, 2])
def test_derivatives_match_fd(orc, fam, which):
    # test_kernels.cpp:122-152 — central FD in the raw parameter, step 1e-6, rel 1e-5
    x = orc.random_matrix(32, 2, 11)
    v = np.random.default_rng(11).standard_normal(32)
    f = orc.FAMILIES[fam]
    p = orc.Params(2, 1.4, 0.8, 0.05)
    step = 1e-6

    def dense_at(raw):
        q = orc.Params(2, 1.4, 0.8, 0.05)
        if which == 0:
            q.log_o = math.log(raw)
        else:
            q.log_ls = q.log_ls.copy()
            q.log_ls[which - 1] = math.log(raw)
        return orc.dense(f, x, q)

    raw0 = p.raw(which)
    fd = (dense_at(raw0 + step) - dense_at(raw0 - step)) / (2 * step)
    want = np.tril(fd) @ v + np.tril(fd, -1).T @ v  # selfadjointView<Lower>
    got = orc.kernel_apply(f, x, p, v, which=which)[:, 0]
    assert np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-12) < 1e-5


def test_outputscale_derivative(orc):
    # test_kernels.cpp:154-164
    x = orc.random_matrix(32, 1, 12)
    p = orc.Params(1, 2.0, 1.0, 0.1)
    v = np.random.default_rng(12).standard_normal(32)
    k0 = orc.dense(orc.RBF, x, p) - 0.1 * np.eye(32)
    want = (2.0 / 2.0) * (k0 @ v)
    got = orc.kernel_apply(orc.RBF, x, p, v, which=0)[:, 0]
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


def test_probe_stream_and_seed_mixing(orc):
    # trace_estimation.hpp:27-36 / common.hpp:93-98: fixed seed reproduces bitwise,
    # entries are +-1/sqrt(n), and mix_seed is SplitMix64.
    z1 = orc.make_probes(100, 3, 17)
    z2 = orc.make_probes(100, 3, 17)
    assert np.array_equal(z1, z2)
    assert np.allclose(np.abs(z1), 0.1)
    assert np.allclose(np.linalg.norm(z1, axis=0), 1.0)
    # SplitMix64 restated independently in Python
    def sm(seed, salt):
        m = (1 << 64) - 1
        z = (seed + 0x9E3779B97F4A7C15 * (salt + 1)) & m
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)
    for s, t in [(17, 1), (0, 0), (2**63 + 5, 0xB2D)]:
        assert orc.mix_seed(s, t) == sm(s, t)
