"""CSV ingestion: gpk_load_csv (C-ABI, host code) against the oracle
restatement of load_csv (oracle/dataset.py; dataset.hpp:155-242, csv.hpp:76-116).

The row order is checked exactly (an id column), which pins the product's
mt19937_64 + uniform_int_distribution shuffle against the independent Python
restatement; values bitwise before standardisation, 1e-12 relative after it.
SPEC items (reference SPEC.md, load_csv): 3-row toy file with split (1,0,0) -> all rows in
train with zero-mean standardised columns; de-standardise(standardise(x)) = x to 1e-12;
non-numeric cell -> parse error naming row/column; constant column -> error naming it."""
import numpy as np
import pytest

import paper_2107_00243_b200 as gk
from oracle import dataset as od


def _write(tmp_path, text, name="d.csv"):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def _table(n, d, seed, target_first=False):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(n, d)) * rng.uniform(0.5, 3, size=d) + rng.normal(size=d)
    y = np.sin(x[:, 0]) + 0.1 * rng.normal(size=n)
    cols = [f"f{j}" for j in range(d)]
    head = ["y"] + cols + ["id"] if target_first else cols + ["id", "y"]
    lines = [",".join(head)]
    for i in range(n):
        vals = [repr(float(v)) for v in x[i]]
        row = [repr(float(y[i]))] + vals + [str(i)] if target_first else vals + [str(i), repr(float(y[i]))]
        lines.append(",".join(row))
    return "\n".join(lines) + "\n"


def _check_same(got: "gk.DataSplits", want: dict, standardized: bool):
    for name in ("train", "validation", "test"):
        g = getattr(got, name)
        wx, wy = want[name]
        assert g.x.shape == wx.shape and g.y.shape == wy.shape, name
        if standardized:
            np.testing.assert_allclose(g.x, wx, rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(g.y, wy, rtol=1e-12, atol=1e-12)
        else:
            assert np.array_equal(g.x, wx) and np.array_equal(g.y, wy), name
    assert got.feature_names == want["names"] and got.target_name == want["target"]
    assert got.standardized == want["standardized"]


def test_mt19937_64_known_answer():
    r = od.MT19937_64()
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042  # [rand.predef]


@pytest.mark.parametrize("n,d,seed,split", [(10, 2, 1, (0.64, 0.16, 0.20)), (257, 5, 42, (0.5, 0.25, 0.25)),
                                            (1000, 3, 2**63 + 7, (0.9, 0.0, 0.1)), (33, 1, 0, (0.3, 0.3, 0.3))])
def test_shuffle_split_matches_oracle_raw(tmp_path, n, d, seed, split):
    path = _write(tmp_path, _table(n, d, seed % 1000))
    sf = gk.SplitFractions(*split)
    got = gk.load_csv(path, "y", standardize=False, split=sf, seed=seed)
    want = od.load_csv(path, "y", standardize=False, split=split, seed=seed)
    _check_same(got, want, False)
    ids = got.train.x[:, -1].astype(int).tolist() + got.validation.x[:, -1].astype(int).tolist() + \
        got.test.x[:, -1].astype(int).tolist()
    assert ids == [int(v) for v in want["order"][:len(ids)]]


@pytest.mark.parametrize("target_first", [False, True])
def test_standardized_matches_oracle(tmp_path, target_first):
    path = _write(tmp_path, _table(500, 4, 3, target_first))
    got = gk.load_csv(path, "y", standardize=True, seed=11)
    want = od.load_csv(path, "y", standardize=True, seed=11)
    _check_same(got, want, True)
    mu, sd, tm, ts = want["stats"]
    np.testing.assert_allclose(got.stats.feature_mean, mu, rtol=1e-13)
    np.testing.assert_allclose(got.stats.feature_std, sd, rtol=1e-13)
    assert abs(got.stats.target_mean - tm) <= 1e-13 * max(1.0, abs(tm))
    assert abs(got.stats.target_std - ts) <= 1e-13 * ts
    # training split: zero mean, unit population variance
    np.testing.assert_allclose(got.train.x.mean(axis=0), 0.0, atol=1e-12)
    np.testing.assert_allclose(got.train.x.std(axis=0), 1.0, rtol=1e-12)


def test_spec_toy_file_all_train(tmp_path):
    path = _write(tmp_path, "a,b,t\n1,10,3\n2,20,5\n4,70,4\n")
    got = gk.load_csv(path, "t", standardize=True, split=gk.SplitFractions(1.0, 0.0, 0.0), seed=5)
    assert got.train.size() == 3 and got.validation.size() == 0 and got.test.size() == 0
    np.testing.assert_allclose(got.train.x.mean(axis=0), 0.0, atol=1e-15)
    assert abs(got.train.y.mean()) <= 1e-15


def test_spec_round_trip(tmp_path):
    path = _write(tmp_path, _table(200, 3, 9))
    raw = gk.load_csv(path, "y", standardize=False, seed=4)
    std = gk.load_csv(path, "y", standardize=True, seed=4)
    for name in ("train", "validation", "test"):
        r, s = getattr(raw, name), getattr(std, name)
        np.testing.assert_allclose(std.stats.invert_x(s.x), r.x, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(std.stats.invert_y(s.y), r.y, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(std.stats.transform_x(r.x), s.x, rtol=1e-12, atol=1e-12)


def test_dataset_invert_c_abi(tmp_path):
    """gpk_dataset_invert (Standardizer::invert_x / invert_y) in place."""
    import ctypes as C

    from paper_2107_00243_b200 import capi
    path = _write(tmp_path, _table(64, 2, 1))
    lib = capi.lib()
    h = C.c_void_p()
    assert lib.gpk_load_csv(path.encode(), b"y", 1, 0.5, 0.25, 0.25, 3, C.byref(h), None, 0) == 0
    raw = gk.load_csv(path, "y", standardize=False, split=gk.SplitFractions(0.5, 0.25, 0.25), seed=3)
    n = C.c_int64()
    d = C.c_int()
    lib.gpk_dataset_shape(h, 2, C.byref(n), C.byref(d))
    x = np.zeros((n.value, d.value), order="F")
    y = np.zeros(n.value)
    dp = C.POINTER(C.c_double)
    lib.gpk_dataset_copy(h, 2, x.ctypes.data_as(dp), n.value, y.ctypes.data_as(dp))
    assert lib.gpk_dataset_invert(h, x.ctypes.data_as(dp), n.value, n.value, y.ctypes.data_as(dp)) == 0
    lib.gpk_dataset_free(h)
    np.testing.assert_allclose(x, raw.test.x, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(y, raw.test.y, rtol=1e-12, atol=1e-12)


def test_format_edge_cases(tmp_path):
    """comments, CRLF, blank lines, whitespace trimming, hex / inf cells parse as std::stod does."""
    text = ("# schema: toy\r\n\r\n a , b ,\tt \r\n# comment\n1,0x1p3,2\n\n 3 ,+.5e1, 7\r\n5,6,1e2\n"
            "2.5,-0,4\n")
    path = _write(tmp_path, text)
    got = gk.load_csv(path, "t", standardize=False, split=gk.SplitFractions(1.0, 0, 0), seed=1)
    want = od.load_csv(path, "t", standardize=False, split=(1.0, 0, 0), seed=1)
    _check_same(got, want, False)
    assert got.feature_names == ["a", "b"]
    assert sorted(got.train.x[:, 1].tolist()) == [-0.0, 5.0, 6.0, 8.0]


def _err(path, target="t", **kw):
    with pytest.raises(gk.InputError) as e:
        gk.load_csv(path, target, **kw)
    with pytest.raises(od.InputError) as w:
        od.load_csv(path, target, **{k: (tuple(vars(v).values()) if k == "split" else v) for k, v in kw.items()})
    assert str(e.value) == str(w.value)
    return str(e.value)


@pytest.mark.parametrize("text,needle", [
    ("a,t\n1,2\n3,x\n", "non-numeric cell 'x' at data row 2, column 2"),
    ("a,t\n1,2\n3,4,\n", "data row 2 has 3 cells, expected 2"),
    ("a,t\n1,2\n3\n", "data row 2 has 1 cells, expected 2"),
    ("a,t\n1,1e999\n", "non-numeric cell '1e999'"),
    ("a,t\n1,2abc\n", "non-numeric cell '2abc'"),
    ("a,t\n1,\n", "non-numeric cell ''"),
    ("1,2\n3,4\n", "has no header row"),
    ("# only a comment\n\n", "is empty"),
    ("a,t\n", "no data rows"),
    ("t\n1\n2\n", "need at least one feature column"),
    ("a,b\n1,2\n", "no column named 't'"),
])
def test_input_errors(tmp_path, text, needle):
    msg = _err(_write(tmp_path, text))
    assert needle in msg


def test_constant_column_and_target_errors(tmp_path):
    msg = _err(_write(tmp_path, "a,b,t\n1,5,1\n2,5,2\n3,5,3\n4,5,4\n"), standardize=True,
               split=gk.SplitFractions(1.0, 0.0, 0.0), seed=0)
    assert "column 'b' is constant on the training split" in msg
    msg = _err(_write(tmp_path, "a,t\n1,5\n2,5\n3,5\n", "c.csv"), standardize=True,
               split=gk.SplitFractions(1.0, 0.0, 0.0), seed=0)
    assert "target column 't' is constant" in msg
    msg = _err(_write(tmp_path, "a,t\n1,5\n2,6\n3,7\n", "e.csv"), standardize=True,
               split=gk.SplitFractions(0.2, 0.0, 0.0), seed=0)
    assert "at least two training rows" in msg
    msg = _err(_write(tmp_path, "a,t\n1,5\n", "f.csv"), split=gk.SplitFractions(0.7, 0.4, 0.0), seed=0)
    assert "split fractions" in msg
    with pytest.raises(gk.InputError, match="cannot open"):
        gk.load_csv(str(tmp_path / "missing.csv"), "t")


def test_first_bad_row_wins_across_parse_threads(tmp_path):
    """The parser splits rows over host threads; the reported error is the first bad row, as in
    the reference's serial loop."""
    n = 40000
    lines = ["a,t"] + [f"{i},{i % 7}" for i in range(n)]
    lines[30001] = "1,oops"
    lines[20001] = "2,3,4"
    path = _write(tmp_path, "\n".join(lines) + "\n")
    with pytest.raises(gk.InputError, match="data row 20001 has 3 cells"):
        gk.load_csv(path, "t")


def test_large_file_matches_oracle(tmp_path):
    path = _write(tmp_path, _table(20000, 6, 17))
    got = gk.load_csv(path, "y", standardize=True, seed=123)
    want = od.load_csv(path, "y", standardize=True, seed=123)
    _check_same(got, want, True)


@pytest.mark.gpu
def test_csv_training_split_through_the_hot_path(tmp_path, orc):
    """load_csv -> train split -> pivoted Cholesky + evaluate_mll on the device, against the
    oracle evaluated on the oracle loader's split (the caller chain of run_training_arm,
    experiments.hpp:403-414)."""
    path = _write(tmp_path, _table(1200, 3, 21))
    got = gk.load_csv(path, "y", standardize=True, seed=8)
    want = od.load_csv(path, "y", standardize=True, seed=8)
    x, y = got.train.x, got.train.y
    xw, yw = want["train"]
    np.testing.assert_allclose(x, xw, rtol=1e-12, atol=1e-12)
    d = x.shape[1]
    n = x.shape[0]
    hp = gk.Hyperparameters.from_raw(d, 1.0, 1.2, 0.05)
    seed = gk.mix_seed(17, 1)
    z = gk.make_probes(n, 6, seed)
    op = gk.KernelOperator(gk.KernelSpec("rbf"), x, hp)
    pc = gk.pivoted_cholesky_with_derivatives(op, 12)
    cfg = gk.MllConfig(gk.CgConfig(200, 1e-8, False, "fp64", 2), True, "fused")
    r = gk.evaluate_mll(y, op, pc, z, cfg)
    ref = orc.evaluate_mll(orc.RBF, np.asfortranarray(xw), orc.Params(d, 1.0, 1.2, 0.05), yw, z.probes, seed=seed,
                           prec="pivchol", rank=12, max_iters=200, rel_tol=1e-8)
    assert abs(r.value - ref["value"]) <= 1e-4 * abs(ref["value"])
    err = np.max(np.abs(r.gradient - ref["gradient"]) / np.maximum(np.abs(ref["gradient"]), 1e-8))
    assert err <= 1e-4
