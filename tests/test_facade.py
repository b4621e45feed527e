"""The C++ facade (include/gpkrylov_cuda.hpp) compiles against the C-ABI (CPU) and, on a
GPU, a C++ caller reproduces the oracle's evaluate_mll (gpu)."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_2107_00243_b200", "lib")


def build(tmp_path):
    exe = str(tmp_path / "facade_test")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), SRC, "-o", exe,
                    "-L" + LIBDIR, "-lgpkrylov_cuda", "-Wl,-rpath," + LIBDIR], check=True)
    return exe


def test_facade_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_facade_cpp_caller_matches_oracle(tmp_path, orc):
    exe = build(tmp_path)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    got = json.loads(out)
    n, d, l = 400, 2, 6
    i = np.arange(n)
    x = np.stack([np.sin(0.37 * i) * 1.5, np.cos(0.11 * i + 0.3)], axis=1)
    y = np.sin(2.0 * x[:, 0]) + 0.3 * x[:, 1]
    p = orc.Params(d, 1.1, 0.8, 0.05)
    seed = orc.mix_seed(17, 1)
    assert got["seed"] == seed
    z = orc.make_probes(n, l, seed)
    want = orc.evaluate_mll(orc.MATERN52, x, p, y, z, seed=seed, prec="pivchol", rank=12, max_iters=400,
                            rel_tol=1e-10)
    ref_piv = orc.pivoted_cholesky(12, family=orc.MATERN52, x=x, p=p)["pivots"]
    assert got["pivots"] == list(ref_piv)
    assert got["value"] == pytest.approx(want["value"], rel=1e-9)
    np.testing.assert_allclose(got["gradient"], want["gradient"], rtol=1e-7, atol=1e-9)
    # SURVEY.md §8(f) through the facade: dense exact mLL, optimize()
    assert got["exact"] == pytest.approx(orc.mll_exact_value(orc.MATERN52, x, p, y), rel=1e-10)
    opt = orc.optimize(orc.MATERN52, x, y, None, None, p, rank=12, probe_count=l, max_iters=400, rel_tol=1e-10,
                       seed=17, method=1, max_steps=3)
    assert got["opt_evals"] == len(opt["evaluations"])
    np.testing.assert_allclose(got["opt_best"], opt["best"], rtol=1e-6, atol=1e-7)


def test_facade_load_csv_matches_oracle(tmp_path):
    """gpkrylov::cuda::load_csv from a compiled C++ caller (host only) against oracle/dataset.py."""
    from oracle import dataset as od

    exe = str(tmp_path / "load_csv_test")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "load_csv_test.cpp"), "-o", exe, "-L" + LIBDIR,
                    "-lgpkrylov_cuda", "-Wl,-rpath," + LIBDIR], check=True)
    rng = np.random.default_rng(5)
    x = rng.normal(size=(150, 4))
    path = tmp_path / "t.csv"
    path.write_text("u,v,target,w\n" + "\n".join(",".join(repr(float(v)) for v in r) for r in x) + "\n")
    got = json.loads(subprocess.run([exe, str(path), "target", "1", "99"], check=True, capture_output=True,
                                    text=True).stdout)
    want = od.load_csv(str(path), "target", standardize=True, seed=99)
    assert got["names"] == ["u", "v", "w"] and got["target"] == "target" and got["standardized"]
    for name in ("train", "validation", "test"):
        wx, wy = want[name]
        g = got[name]
        assert g["n"] == len(wy)
        np.testing.assert_allclose(np.array(g["x"]).reshape(3, -1).T, wx, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(g["y"], wy, rtol=1e-12, atol=1e-12)
    bad = tmp_path / "b.csv"
    bad.write_text("a,target\n1,2\n3,zz\n")
    r = subprocess.run([exe, str(bad), "target", "1", "1"], capture_output=True, text=True)
    assert r.returncode == 1
    assert "non-numeric cell 'zz' at data row 2, column 2" in r.stdout
