"""Shared test fixtures (restating proj/tests/support.hpp)."""
import numpy as np


def random_spd(n, seed, lo=0.5, hi=4.0):
    """support.hpp:29-37 restated: Q (orthogonal, QR of a Gaussian matrix) diag(U[lo,hi]) Q^T."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = rng.uniform(lo, hi, n)
    m = (q * lam) @ q.T
    return 0.5 * (m + m.T)
