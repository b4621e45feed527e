"""Pins the CPU oracle's pcg_solve / SLQ / probes to the reference's own
known-answer tests (proj/tests/test_krylov.cpp)."""
import numpy as np
import pytest

from helpers import random_spd


def mt19937_64(seed, count):
    """Independent pure-Python MT19937-64 (the standardized std::mt19937_64 stream)."""
    w, n, m, r = 64, 312, 156, 31
    a, u, d, s, b, t, c, l, f = (0xB5026F5AA96619E9, 29, 0x5555555555555555, 17, 0x71D67FFFEDA60000, 37,
                                 0xFFF7EEE000000000, 43, 6364136223846793005)
    mask = (1 << 64) - 1
    mt = [0] * n
    mt[0] = seed & mask
    for i in range(1, n):
        mt[i] = (f * (mt[i - 1] ^ (mt[i - 1] >> (w - 2))) + i) & mask
    lower = (1 << r) - 1
    upper = (~lower) & mask
    idx = n
    out = []
    for _ in range(count):
        if idx >= n:
            for i in range(n):
                x = (mt[i] & upper) | (mt[(i + 1) % n] & lower)
                xa = x >> 1
                if x & 1:
                    xa ^= a
                mt[i] = mt[(i + m) % n] ^ xa
            idx = 0
        y = mt[idx]
        idx += 1
        y ^= (y >> u) & d
        y ^= (y << s) & b
        y ^= (y << t) & c
        y ^= y >> l
        out.append(y & mask)
    return out


def test_probe_stream_is_mt19937_64(orc):
    # make_probes (trace_estimation.hpp:27-36): z(i,c) = (rng() & 1) ? +1/sqrt(n) : -1/sqrt(n), c outer, i inner
    n, l, seed = 40, 3, orc.mix_seed(17, 1)
    bits = mt19937_64(seed, n * l)
    want = np.array([1.0 if b & 1 else -1.0 for b in bits]).reshape((n, l), order="F") / np.sqrt(n)
    assert np.array_equal(orc.make_probes(n, l, seed), want)
    # the C++ standard's check value for the default seed (10000th draw)
    assert mt19937_64(5489, 10000)[-1] == 9981545732273789042


def test_identity_one_iteration(orc):
    # test_krylov.cpp:16-25
    b = np.random.default_rng(21).standard_normal(16)
    r = orc.pcg_dense(np.eye(16), b, max_iters=50, rel_tol=1e-10)
    assert r["converged"] and r["iterations"] == 1
    assert np.linalg.norm(r["solution"] - b) < 1e-14


def test_diagonal_exact(orc):
    # test_krylov.cpp:27-35
    r = orc.pcg_dense(np.diag([1.0, 2.0]), np.array([1.0, 2.0]), max_iters=10, rel_tol=1e-12)
    assert r["iterations"] <= 2
    assert np.linalg.norm(r["solution"] - 1.0) < 1e-12


def test_perfect_preconditioner(orc):
    # test_krylov.cpp:37-51
    m = random_spd(32, 22)
    b = np.random.default_rng(22).standard_normal(32)
    r = orc.pcg_dense(m, b, prec="exact", pmat=m, max_iters=32, rel_tol=1e-10)
    assert r["converged"] and r["iterations"] <= 2
    assert np.linalg.norm(m @ r["solution"] - b) / np.linalg.norm(b) < 1e-9


def test_matches_dense_solve(orc):
    # test_krylov.cpp:53-62
    m = random_spd(64, 23)
    b = np.random.default_rng(23).standard_normal(64)
    r = orc.pcg_dense(m, b, max_iters=200, rel_tol=1e-12)
    want = np.linalg.solve(m, b)
    assert np.linalg.norm(r["solution"] - want) / np.linalg.norm(want) < 1e-9
    assert len(r["residual_history"]) == r["iterations"]


def test_a_norm_monotone(orc):
    # test_krylov.cpp:64-81
    m = random_spd(48, 24, 0.1, 10.0)
    b = np.random.default_rng(24).standard_normal(48)
    xs = np.linalg.solve(m, b)
    prev = np.inf
    for k in range(1, 21):
        e = orc.pcg_dense(m, b, max_iters=k, rel_tol=1e-15)["solution"] - xs
        an = np.sqrt(e @ m @ e)
        assert an <= prev * (1 + 1e-10)
        prev = an


def test_ritz_values_and_slq_exactness(orc):
    # test_krylov.cpp:83-111 and SPEC acceptance #4
    m = random_spd(64, 25, 0.5, 8.0)
    z = orc.make_probes(64, 1, 99)[:, 0]
    r = orc.pcg_dense(m, z, max_iters=64, rel_tol=1e-15, collect=True)
    assert len(r["tdiag"]) == r["iterations"]
    assert r["tdiag"].min() > 0
    if r["iterations"] == 64:
        t = np.diag(r["tdiag"]) + np.diag(r["tsub"], 1) + np.diag(r["tsub"], -1)
        assert np.max(np.abs(np.linalg.eigvalsh(t) - np.linalg.eigvalsh(m))) < 1e-7
    q = orc.slq(r["tdiag"], r["tsub"])
    w, v = np.linalg.eigh(m)
    want = z @ (v * np.log(w)) @ v.T @ z
    assert q["value"] == pytest.approx(want, rel=1e-8)
    # oracle's dense matrix log agrees as well (oracle.hpp:72-77)
    _, _, _, ml = orc.dense_spd(m, want_log=True)
    assert z @ ml @ z == pytest.approx(want, rel=1e-10)


def test_slq_exactness_20_probes(orc):
    # SPEC acceptance #4: m = n, n = 32, 20 probes, rel 1e-8
    m = random_spd(32, 44, 0.5, 8.0)
    w, v = np.linalg.eigh(m)
    logm = (v * np.log(w)) @ v.T
    zs = orc.make_probes(32, 20, 7)
    for i in range(20):
        r = orc.pcg_dense(m, zs[:, i], max_iters=32, rel_tol=1e-15, collect=True)
        assert orc.slq(r["tdiag"], r["tsub"])["value"] == pytest.approx(zs[:, i] @ logm @ zs[:, i], rel=1e-8)


def test_slq_clamps_and_weights(orc):
    # trace_estimation.hpp:97-107: weights sum to 1 (first eigvec row), floor 1e-12 max|node|
    t = orc.slq(np.array([2.0, 3.0, 1e-20]), np.array([0.5, 1e-30]))
    assert t["weights"].sum() == pytest.approx(1.0, rel=1e-14)
    assert t["clamped"] == 1
    assert orc.slq(np.array([]), np.array([]))["value"] == 0.0


def test_breakdown_raises(orc):
    # test_krylov.cpp:113-120
    with pytest.raises(orc.SolverError, match="pcg_solve: breakdown at iteration"):
        orc.pcg_dense(np.diag([1.0, -2.0, 3.0]), np.ones(3), max_iters=10, rel_tol=1e-10)


def test_config_validation(orc):
    # test_krylov.cpp:122-132
    with pytest.raises(orc.InputError):
        orc.pcg_dense(np.eye(4), np.ones(4), max_iters=0, rel_tol=0.5)
    with pytest.raises(orc.InputError):
        orc.pcg_dense(np.eye(4), np.ones(4), max_iters=5, rel_tol=0.0)


def test_batched_equals_independent_bitwise(orc):
    # test_krylov.cpp:134-151 (batched_pcg contract) on the kernel operator
    x = orc.random_matrix(128, 2, 26)
    p = orc.Params(2, 1.0, 0.7, 0.05)
    b = orc.random_matrix(128, 8, 260)
    sol, it, cv = orc.pcg_kernel(orc.RBF, x, p, b, rank=8, max_iters=300, rel_tol=1e-6)
    k = orc.dense(orc.RBF, x, p)
    for c in range(8):
        s1, i1, _ = orc.pcg_kernel(orc.RBF, x, p, b[:, c], rank=8, max_iters=300, rel_tol=1e-6)
        assert i1[0] == it[c]
        assert np.array_equal(s1[:, 0], sol[:, c])
        want = np.linalg.solve(k, b[:, c])
        assert np.linalg.norm(sol[:, c] - want) / np.linalg.norm(want) < 1e-5


def test_batched_identity_basis(orc):
    # test_krylov.cpp:153-162
    for c in range(4):
        r = orc.pcg_dense(np.eye(16), np.eye(16)[:, c], max_iters=8, rel_tol=1e-12)
        assert r["iterations"] == 1
        assert np.linalg.norm(r["solution"] - np.eye(16)[:, c]) < 1e-15


def test_preconditioning_does_not_increase_iterations(orc):
    # test_krylov.cpp:164-178 — 1-d RBF n=1000, rank-32 pivoted Cholesky
    xb = orc.random_matrix(2000, 1, 27)  # same gen stream: x then b
    x, b = xb[:1000], xb[1000:, 0]
    p = orc.Params(1, 1.0, 0.5, 1e-2)
    _, ip, _ = orc.pcg_kernel(orc.RBF, x, p, b, rank=-1, max_iters=1000, rel_tol=1e-6)
    _, iq, cq = orc.pcg_kernel(orc.RBF, x, p, b, rank=32, max_iters=1000, rel_tol=1e-6)
    assert iq[0] <= ip[0]
    assert cq[0] == 1


def test_zero_rhs(orc):
    # test_krylov.cpp:180-188
    r = orc.pcg_dense(np.eye(8), np.zeros(8), max_iters=10, rel_tol=1e-10)
    assert r["converged"] and r["iterations"] == 0 and np.linalg.norm(r["solution"]) == 0.0
