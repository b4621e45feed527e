"""CPU oracle for CSV dataset ingestion — TEST INFRASTRUCTURE ONLY (the checker of
gpk_load_csv; never imported by the product package).

Pure-Python restatement of the reference's
  * read_csv_table / split_csv_line   (/root/reference/proj/include/gpkrylov/csv.hpp:76-116)
  * load_csv                          (/root/reference/proj/include/gpkrylov/dataset.hpp:155-242)
  * Standardizer                      (dataset.hpp:87-101)
and of the two third-party algorithms the reference takes from the C++ standard
library (libstdc++ of GCC 13.3, the toolchain here):
  * std::mt19937_64 — the Mersenne Twister MT19937-64 (the standard's parameters); pinned
    by the standard's own known answer (10000th output of the default seed 5489 is
    9981545732273789042, [rand.predef]);
  * std::uniform_int_distribution<long>(0, i) over a 64-bit engine — libstdc++'s
    downscaling by Lemire's nearly divisionless method with 128-bit products
    (bits/uniform_int_dist.h, _S_nd);
  * std::stod — strtod's decimal / hex / inf / nan grammar, the whole cell consumed,
    out-of-range results (overflow, underflow to zero) rejected.
Small inputs only (pure-Python loops).
"""
from __future__ import annotations

import math
import re

import numpy as np

M64 = (1 << 64) - 1


class InputError(ValueError):
    pass


class MT19937_64:
    """std::mt19937_64 (w=64, n=312, m=156, r=31)."""
    N, M = 312, 156
    A = 0xB5026F5AA96619E9
    UPPER, LOWER = (~((1 << 31) - 1)) & M64, (1 << 31) - 1

    def __init__(self, seed: int = 5489):
        mt = [seed & M64]
        for i in range(1, self.N):
            mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & M64)
        self.mt, self.i = mt, self.N

    def _twist(self):
        mt, n, m = self.mt, self.N, self.M
        for k in range(n):
            y = (mt[k] & self.UPPER) | (mt[(k + 1) % n] & self.LOWER)
            mt[k] = mt[(k + m) % n] ^ (y >> 1) ^ (self.A if y & 1 else 0)
        self.i = 0

    def __call__(self) -> int:
        if self.i >= self.N:
            self._twist()
        z = self.mt[self.i]
        self.i += 1
        z ^= (z >> 29) & 0x5555555555555555
        z ^= (z << 17) & 0x71D67FFFEDA60000
        z ^= (z << 37) & 0xFFF7EEE000000000
        z ^= z >> 43
        return z & M64


def uniform_int(rng: MT19937_64, a: int, b: int) -> int:
    """std::uniform_int_distribution<long>(a, b)(rng) in libstdc++ (64-bit engine: _S_nd)."""
    rng_range = (b - a) & M64
    if rng_range == M64:
        return (rng() + a) & M64
    r = rng_range + 1
    prod = rng() * r
    low = prod & M64
    if low < r:
        threshold = ((-r) & M64) % r
        while low < threshold:
            prod = rng() * r
            low = prod & M64
    return a + (prod >> 64)


_NUM = re.compile(r"[ \t\n\v\f\r]*[+-]?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|"
                  r"\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?|[iI][nN][fF](?:[iI][nN][iI][tT][yY])?|"
                  r"[nN][aA][nN](?:\([0-9A-Za-z_]*\))?)")


def stod_whole(cell: str):
    """std::stod(cell, &pos) with pos == cell.size() (dataset.hpp:121-132); None when rejected."""
    m = _NUM.fullmatch(cell)
    if not m:
        return None
    s = cell.strip(" \t\n\v\f\r")
    body = s.lstrip("+-").lower()
    if body.startswith("0x"):
        mant, _, exp = body[2:].partition("p")
        ip, _, fp = mant.partition(".")
        v = float(int((ip + fp) or "0", 16)) * 2.0 ** (int(exp or "0") - 4 * len(fp))
        v = -v if s.startswith("-") else v
    else:
        sign = -1.0 if s.startswith("-") else 1.0
        v = math.nan if body.startswith("nan") else sign * math.inf if body.startswith("inf") else float(s)
    finite_literal = not re.search(r"inf|nan", body)
    if finite_literal and (math.isinf(v) or (v == 0.0 and re.search(r"[1-9]", body.split("e")[0].split("p")[0]))):
        return None  # ERANGE -> std::out_of_range
    return v


def split_csv_line(line: str) -> list:
    """csv.hpp:76-89 (getline on ',' semantics; cells trimmed of ' \\t\\r')."""
    cells = line.split(",")
    if cells and cells[-1] == "":  # getline yields no final empty field ...
        cells.pop()
    out = [c.strip(" \t\r") for c in cells]
    if line.endswith(","):  # ... the reference appends it explicitly
        out.append("")
    return out


def read_csv_table(path: str):
    """csv.hpp:91-116 -> (columns, rows)."""
    try:
        text = open(path, "rb").read().decode("latin-1")
    except OSError:
        raise InputError("read_csv_table: cannot open " + path)
    columns, rows, have = [], [], False
    parts = text.split("\n")
    if parts and parts[-1] == "":
        parts.pop()
    for line in parts:
        if line.endswith("\r"):
            line = line[:-1]
        if not line or line[0] == "#":
            continue
        cells = split_csv_line(line)
        if not have:
            columns, have = cells, True
        else:
            rows.append(cells)
    return columns, rows


def llround(v: float) -> int:
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def load_csv(path: str, target_column: str, standardize: bool = True, split=(0.64, 0.16, 0.20), seed: int = 0):
    """dataset.hpp:155-242.  Returns dict(train=(x, y), validation=..., test=..., stats=..., names=...)."""
    columns, rows = read_csv_table(path)
    if not columns:
        raise InputError("load_csv: " + path + " is empty")
    if all(stod_whole(c) is not None for c in columns):
        raise InputError("load_csv: " + path + " has no header row")
    ft, fv, fs = split
    if not (ft >= 0 and fv >= 0 and fs >= 0 and ft + fv + fs <= 1.0 + 1e-9):
        raise InputError("load_csv: split fractions must be nonnegative and sum to at most 1")
    if target_column not in columns:
        raise InputError("CsvTable: no column named '" + target_column + "'")
    target = columns.index(target_column)
    n = len(rows)
    if n < 1:
        raise InputError("load_csv: no data rows in " + path)
    ncols = len(columns)
    d = ncols - 1
    if d < 1:
        raise InputError("load_csv: need at least one feature column")
    x = np.zeros((n, d))
    y = np.zeros(n)
    for i, row in enumerate(rows):
        if len(row) != ncols:
            raise InputError(f"load_csv: data row {i + 1} has {len(row)} cells, expected {ncols}")
        fc = 0
        for c, cell in enumerate(row):
            v = stod_whole(cell)
            if v is None:
                raise InputError(f"load_csv: non-numeric cell '{cell}' at data row {i + 1}, column {c + 1}")
            if c == target:
                y[i] = v
            else:
                x[i, fc] = v
                fc += 1
    order = list(range(n))
    rng = MT19937_64(seed)
    for i in range(n - 1, 0, -1):  # dataset.hpp:185-191
        j = uniform_int(rng, 0, i)
        order[i], order[j] = order[j], order[i]
    n_train = min(n, llround(ft * n))
    n_val = min(n - n_train, llround(fv * n))
    n_test = min(n - n_train - n_val, llround(fs * n))
    idx = np.array(order, dtype=np.int64)
    parts = {}
    for name, b, c in (("train", 0, n_train), ("validation", n_train, n_val), ("test", n_train + n_val, n_test)):
        parts[name] = (x[idx[b:b + c]], y[idx[b:b + c]])
    names = [columns[c] for c in range(ncols) if c != target]
    out = dict(parts, order=order, names=names, target=target_column, standardized=False,
               stats=(np.zeros(d), np.ones(d), 0.0, 1.0))
    if standardize:
        xt, yt = parts["train"]
        if len(yt) < 2:
            raise InputError("load_csv: standardization needs at least two training rows")
        mu = xt.mean(axis=0)
        sd = np.sqrt(((xt - mu) ** 2).sum(axis=0) / len(yt))
        for j in range(d):
            if not sd[j] > 1e-12:
                raise InputError(f"load_csv: column '{names[j]}' is constant on the training split; "
                                 "cannot standardize")
        tm = yt.mean()
        ts = math.sqrt(((yt - tm) ** 2).sum() / len(yt))
        if not ts > 1e-12:
            raise InputError(f"load_csv: target column '{target_column}' is constant on the training split; "
                             "cannot standardize")
        for name in ("train", "validation", "test"):
            px, py = parts[name]
            out[name] = ((px - mu) / sd, (py - tm) / ts)
        out["standardized"] = True
        out["stats"] = (mu, sd, tm, ts)
    return out
