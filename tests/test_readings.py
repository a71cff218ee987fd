"""CPU checks of algorithmic readings in DESIGN.md that the GPU path relies on
(not of the oracle: these run the numpy models in scripts/)."""
import importlib.util
import os

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "scripts", name + ".py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_r22_three_term_z_recurrence_keeps_cg_accuracy():
    """R22: the three-term z recurrence with two-term p/x updates reproduces
    Hestenes-Stiefel CG (iterates, iteration count, attainable accuracy),
    while a three-term x recurrence does not keep the true residual."""
    cr = _load("cg_recurrences")
    rng = np.random.default_rng(1)
    n = 3000
    k = rng.uniform(0.5, 2.0, n + 1)
    A = sp.diags([-k[1:-1], k[:-1] + k[1:], -k[1:-1]], [-1, 0, 1]).tocsr()
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    d = A.diagonal()
    bn = np.linalg.norm(b)
    xh, kh = cr.hs(A, b, x0, d, 1e-10, 20 * n)
    x2, k2 = cr.cg3(A, b, x0, d, 1e-10, 20 * n, True)
    x3, k3 = cr.cg3(A, b, x0, d, 1e-10, 20 * n, False)
    rh = np.linalg.norm(b - A @ xh) / bn
    r2 = np.linalg.norm(b - A @ x2) / bn
    r3 = np.linalg.norm(b - A @ x3) / bn
    assert abs(k2 - kh) <= 10, (kh, k2)
    assert np.linalg.norm(x2 - xh) <= 1e-8 * np.linalg.norm(xh)
    assert r2 <= 3 * rh + 1e-10, (rh, r2)
    assert r3 > 10 * rh, (rh, r3)  # why x stays on the two-term update
