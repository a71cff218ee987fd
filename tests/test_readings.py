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


def test_r25_momentum_guess_is_the_previous_intermediate_velocity():
    """R25 (oracle): the momentum solves of a step start from the previous
    step's u*, v*.  Started from u^n instead, the same systems reach the same
    solution (to the stopping point) but from a larger initial residual: the
    projected u^n differs from u* by the pressure-gradient correction of
    Eq. 21, the previous u* only by one step's change."""
    import sys
    sys.path.insert(0, ROOT)
    from oracle import Params, initial_state, step
    from oracle.krylov import cg
    from oracle.step import ch_system, momentum_systems
    from workloads import initial_fields
    prm = Params(rtol=1e-12)
    st = initial_state(initial_fields(32, 32, seed=1))
    assert st.us is None and st.guess_uv()[0] is st.u
    for _ in range(3):
        st, _ = step(st, prm)
    assert st.us is not None
    _, _, phs = ch_system(st, prm)
    (Au, bu), _ = momentum_systems(st, phs, prm)
    dinv = 1.0 / Au.diagonal()
    r_prev = np.linalg.norm(bu - Au @ st.us.ravel())
    r_un = np.linalg.norm(bu - Au @ st.u.ravel())
    assert r_prev < 0.1 * r_un, (r_prev, r_un)
    x1, k1 = cg(Au, bu, st.us.ravel(), dinv, 1e-12, 10 ** 5)
    x2, k2 = cg(Au, bu, st.u.ravel(), dinv, 1e-12, 10 ** 5)
    assert k1 < k2, (k1, k2)
    assert np.linalg.norm(x1 - x2) <= 1e-8 * np.linalg.norm(x2)
