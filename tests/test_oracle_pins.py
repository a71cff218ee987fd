"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: the paper's printed numbers,
exact discrete eigenpairs, closed-form one-step amplification factors,
manufactured solutions (convergence order), conservation laws, dense direct
solves, or the independent brute-force loop formulation (oracle/brute.py).
"""
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import assemble as asm
from oracle import brute
from oracle import explicit as ex
from oracle.krylov import bicgstab, cg, gmres
from oracle.params import Params, nondimensionalise
from oracle.step import (State, ch_system, initial_state, momentum_systems,
                         nutrient_system, step)
from workloads import initial_fields

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_kv(name):
    out = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if line:
            k, v = line.split("=")
            out[k.strip()] = float(v)
    return out


def _grid(nx, ny):
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    return np.meshgrid(x, y)


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


# ------------------------------------------------------------ paper's numbers
def test_table1_to_section5():
    """§5's printed dimensionless values follow from Table 1 via Eq. 15."""
    g = _golden_kv("paper_parameters.txt")
    nd = nondimensionalise(t0=g["t0"], h0=g["h0"], rho0=g["rho"], eta_s=g["eta_s"],
                           eta_n=g["eta_n"], D=g["D"], mu_dim=g["mu"], A_dim=g["A"])
    assert nd["Re_s"] == pytest.approx(g["Re_s_printed"], rel=2e-3)
    assert nd["Re_n"] == pytest.approx(g["Re_n_printed"], rel=3e-3)
    assert nd["Ds"] == pytest.approx(g["Ds_printed"], rel=1e-12)
    assert nd["mu"] == pytest.approx(g["mu_printed"], rel=1e-12)
    assert nd["A"] == pytest.approx(g["A_printed"], rel=1e-12)
    p = Params()
    for k in ("Re_s", "Re_n", "Lambda", "Gamma1", "Gamma2", "Ds", "mu", "Kc", "A"):
        assert getattr(p, k) == g[k + "_printed"], k


def test_listing3_laplacian_row():
    """Interior row of -h^2 Delta_h equals Listing 3's vals (4, -1, -1, -1, -1)."""
    nx = ny = 8
    A = -asm.lap(nx, ny, "mirror") / (nx * nx)
    j, i = 4, 3
    row = A.getrow(j * nx + i).toarray().ravel()
    for line in open(os.path.join(GOLDEN, "listing3_laplacian.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        di, dj, val = line.split()
        assert row[(j + int(dj)) * nx + (i + int(di))] == pytest.approx(float(val))
    assert np.count_nonzero(row) == 5


def test_periodic_wrap_listing3():
    """'i-1=-1 ... maps to the column corresponding to i=nx-1'."""
    nx, ny = 6, 5
    A = asm.lap(nx, ny, "mirror")
    row = A.getrow(2 * nx + 0).toarray().ravel()
    assert row[2 * nx + nx - 1] == pytest.approx(nx * nx)


# ----------------------------------------------------- brute-force agreement
@pytest.mark.parametrize("nx,ny", [(7, 5), (6, 9)])
def test_assembled_matches_bruteforce(nx, ny):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((ny, nx))
    phis = 0.3 + 0.2 * rng.random((ny, nx))
    prm = Params(Lambda=0.7, Gamma1=1.3, dt=0.1)
    assert _rel(asm.lap(nx, ny) @ x.ravel(), brute.lap(x)) < 1e-13
    Mx, My = ex.mobility_faces(phis, prm.Lambda)
    A = asm.ch_matrix(nx, ny, prm.dt, prm.Gamma1, Mx, My)
    assert _rel(A @ x.ravel(), brute.ch_apply(phis, x, prm.dt, prm.Gamma1, prm.Lambda)) < 1e-13
    bx, by = ex.pressure_faces(phis, 2.0, 1.0)
    assert _rel(asm.poisson_matrix(nx, ny, bx, by) @ x.ravel(),
                brute.poisson_apply(phis, x, 2.0, 1.0)) < 1e-13
    a = 1.0 + rng.random((ny, nx))
    assert _rel(asm.u_matrix(nx, ny, a) @ x.ravel(), brute.u_apply(a, x)) < 1e-13
    xv = x.copy()
    xv[0] = 0.0
    assert _rel(asm.v_matrix(nx, ny, a) @ xv.ravel(), brute.v_apply(a, xv)) < 1e-13
    u = rng.standard_normal((ny, nx))
    v = rng.standard_normal((ny, nx))
    v[0] = 0.0
    assert _rel(ex.divergence(u, v), brute.divergence(u, v)) < 1e-13
    D = asm.mac_div(nx, ny)
    assert _rel(D @ np.concatenate([u.ravel(), v.ravel()]), brute.divergence(u, v)) < 1e-13
    assert _rel(ex.advection(phis, u, v), brute.advection(phis, u, v)) < 1e-13
    cu, cv = brute.convective(u, v, 0.7)
    assert _rel(ex.convective_u(u, v, 0.7), cu) < 1e-13
    assert _rel(ex.convective_v(u, v), cv) < 1e-13
    rx, ry = brute.phase_stress(phis, 2.5)
    Rx, Ry = ex.phase_stress(phis, 2.5)
    assert _rel(Rx, rx) < 1e-13 and _rel(Ry, ry) < 1e-13


def test_mac_poisson_is_div_beta_grad():
    """-D diag(beta) G == poisson_matrix (the projection is exact, Eq. 20-21)."""
    nx, ny = 7, 6
    rng = np.random.default_rng(1)
    phi = rng.random((ny, nx))
    bx, by = ex.pressure_faces(phi, 1.7, 0.9)
    beta = np.concatenate([bx.ravel(), by[:ny].ravel()])
    lhs = -asm.mac_div(nx, ny) @ sp.diags(beta) @ asm.mac_grad(nx, ny)
    assert abs(lhs - asm.poisson_matrix(nx, ny, bx, by)).max() < 1e-9 * nx * nx
    # gradient is minus the adjoint of the divergence on interior faces
    G = asm.mac_grad(nx, ny).toarray()
    DT = asm.mac_div(nx, ny).toarray().T
    inner = np.r_[np.arange(nx * ny), nx * ny + np.arange(nx, nx * ny)]
    assert np.allclose(G[inner], -DT[inner])


# --------------------------------------------------------- exact eigenpairs
@pytest.mark.parametrize("k,l", [(1, 1), (2, 3), (0, 4)])
def test_laplacian_mirror_eigenpair(k, l):
    nx, ny = 12, 10
    X, Y = _grid(nx, ny)
    e = np.cos(2 * np.pi * k * X) * np.cos(np.pi * l * Y)
    lam = -(4 * nx * nx) * np.sin(np.pi * k / nx) ** 2 - (4 * ny * ny) * np.sin(np.pi * l / (2 * ny)) ** 2
    assert _rel(asm.lap(nx, ny) @ e.ravel(), lam * e.ravel()) < 1e-12


@pytest.mark.parametrize("k,l", [(1, 1), (3, 2)])
def test_laplacian_u_and_v_eigenpairs(k, l):
    nx, ny = 10, 12
    X, Y = _grid(nx, ny)
    lam = -(4 * nx * nx) * np.sin(np.pi * k / nx) ** 2 - (4 * ny * ny) * np.sin(np.pi * l / (2 * ny)) ** 2
    eu = np.cos(2 * np.pi * k * (X - 0.5 / nx)) * np.sin(np.pi * l * Y)   # u-face points
    assert _rel(asm.lap(nx, ny, "odd") @ eu.ravel(), lam * eu.ravel()) < 1e-12
    Yf = np.arange(ny)[:, None] / ny * np.ones((1, nx))                    # v-face points
    ev = np.cos(2 * np.pi * k * X) * np.sin(np.pi * l * Yf)
    got = asm.lap(nx, ny, "vface") @ ev.ravel()
    assert _rel(got.reshape(ny, nx)[1:], (lam * ev)[1:]) < 1e-12


# ------------------------------------------------- closed-form one-step pins
def test_ch_step_closed_form_amplification():
    """phi^{n-1} = phi0 + 3 d e, phi^n = phi0 + d e  =>  phi* = phi0 (constant),
    L_M F'(phi*) = 0, and the CN step multiplies the eigenmode e by
    (1/dt - G1/2 L phi0 lam^2)/(1/dt + G1/2 L phi0 lam^2) exactly."""
    nx, ny = 16, 16
    X, Y = _grid(nx, ny)
    k, l = 1, 2
    e = np.cos(2 * np.pi * k * X) * np.cos(np.pi * l * Y)
    lam = -(4 * nx * nx) * np.sin(np.pi * k / nx) ** 2 - (4 * ny * ny) * np.sin(np.pi * l / (2 * ny)) ** 2
    phi0, d = 0.3, 1e-3
    prm = Params(Lambda=0.1, eps=0.0, rtol=1e-14)
    z = np.zeros((ny, nx))
    st = State(phi=phi0 + d * e, phi_prev=phi0 + 3 * d * e, c=np.ones((ny, nx)), u=z, v=z, p=z)
    A, b, phs = ch_system(st, prm)
    assert np.ptp(phs) < 1e-15
    x, _ = bicgstab(A, b, phs.ravel(), 1.0 / A.diagonal(), 1e-14, 1000)
    q = 0.5 * prm.Gamma1 * prm.Lambda * phi0 * lam ** 2
    g = (1 / prm.dt - q) / (1 / prm.dt + q)
    assert 0.1 < g < 0.95                      # the pin is non-trivial
    assert _rel(x, phi0 + d * g * e.ravel()) < 1e-13


def test_nutrient_step_closed_form():
    nx, ny = 12, 8
    X, Y = _grid(nx, ny)
    e = np.cos(2 * np.pi * X) * np.cos(np.pi * Y)
    lam = -(4 * nx * nx) * np.sin(np.pi / nx) ** 2 - (4 * ny * ny) * np.sin(np.pi / (2 * ny)) ** 2
    phi0, c0, d = 0.3, 0.8, 0.05
    prm = Params(dt=1e-3)
    z = np.zeros((ny, nx))
    st = State(phi=np.full((ny, nx), phi0), phi_prev=np.full((ny, nx), phi0),
               c=c0 + d * e, u=z, v=z, p=z)
    A, b = nutrient_system(st, st.phi, prm)
    x, _ = cg(A, b, st.c.ravel(), 1 / A.diagonal(), 1e-14, 1000)
    s = 1 - phi0
    K = prm.Ds * s
    g0 = (s / prm.dt - prm.A * phi0 / 2) / (s / prm.dt + prm.A * phi0 / 2)
    g1 = (s / prm.dt - prm.A * phi0 / 2 + K * lam / 2) / (s / prm.dt + prm.A * phi0 / 2 - K * lam / 2)
    assert _rel(x, (c0 * g0 + d * g1 * e).ravel()) < 1e-13


def test_momentum_shear_mode_closed_form_full_step():
    """x-independent shear mode u = d sin(pi l y), v = 0, uniform phi, lid 0:
    convection and R vanish, D u* = 0 so p = 0, and the full step multiplies
    the mode by (a + lam/2)/(a - lam/2), a = 1/(nu dt)."""
    nx, ny = 8, 16
    X, Y = _grid(nx, ny)
    l = 1
    e = np.sin(np.pi * l * Y)
    lam = -(4 * ny * ny) * np.sin(np.pi * l / (2 * ny)) ** 2
    phi0 = 0.2
    prm = Params(lid_u=0.0, eps=0.0, A=0.0, Re_n=1.0, Re_s=0.5, dt=1e-3, rtol=1e-14)
    nu = phi0 / prm.Re_n + (1 - phi0) / prm.Re_s
    a = 1 / (nu * prm.dt)
    z = np.zeros((ny, nx))
    d = 0.1
    st = State(phi=np.full((ny, nx), phi0), phi_prev=np.full((ny, nx), phi0),
               c=np.ones((ny, nx)), u=d * e, v=z.copy(), p=z.copy())
    new, info = step(st, prm)
    assert _rel(new.u, d * e * (a + lam / 2) / (a - lam / 2)) < 1e-12
    assert np.abs(new.v).max() < 1e-14 and np.abs(new.p).max() < 1e-14
    assert np.abs(new.phi - phi0).max() < 1e-14


def test_couette_is_exact_steady_state():
    """u = U0 y (linear shear under the lid, Eq. 22) is reproduced exactly."""
    nx, ny = 8, 12
    X, Y = _grid(nx, ny)
    prm = Params(lid_u=0.1, eps=0.0, A=0.0, dt=1e-3, rtol=1e-14)
    z = np.zeros((ny, nx))
    st = State(phi=np.full((ny, nx), 0.25), phi_prev=np.full((ny, nx), 0.25),
               c=np.ones((ny, nx)), u=0.1 * Y, v=z.copy(), p=z.copy())
    new, _ = step(st, prm)
    assert _rel(new.u, 0.1 * Y) < 1e-12
    assert np.abs(new.v).max() < 1e-12


def test_uniform_state_is_fixed_point():
    nx, ny = 9, 7
    z = np.zeros((ny, nx))
    prm = Params(lid_u=0.0, eps=0.0, A=0.0)
    st = State(phi=np.full((ny, nx), 0.4), phi_prev=np.full((ny, nx), 0.4),
               c=np.full((ny, nx), 0.7), u=z, v=z, p=z)
    new, _ = step(st, prm)
    for f in ("phi", "c", "u", "v", "p"):
        ref = getattr(st, f)
        assert np.abs(getattr(new, f) - ref).max() <= 1e-15 * max(1.0, np.abs(ref).max()), f


def test_pressure_poisson_eigen_solution():
    nx, ny = 16, 12
    X, Y = _grid(nx, ny)
    e = np.cos(2 * np.pi * X) * np.cos(np.pi * 2 * Y)
    lam = -(4 * nx * nx) * np.sin(np.pi / nx) ** 2 - (4 * ny * ny) * np.sin(np.pi * 2 / (2 * ny)) ** 2
    bx, by = ex.pressure_faces(np.zeros((ny, nx)), 1.0, 1.0)
    A = asm.poisson_matrix(nx, ny, bx, by)
    b = -lam * e.ravel() + 3.0          # constant part removed by the null-space projection
    p, _ = cg(A, b, np.zeros(nx * ny), 1 / A.diagonal(), 1e-13, 2000, nullspace=True)
    assert _rel(p, e.ravel()) < 1e-11
    assert abs(p.mean()) < 1e-14


# --------------------------------------------------------- MMS convergence
def _mms_error(n, which):
    import sympy as syp
    xs, ys = syp.symbols("x y")
    s = syp.cos(2 * syp.pi * xs) * syp.cos(syp.pi * ys)
    K = 1 + syp.Rational(1, 2) * syp.sin(2 * syp.pi * xs) * syp.cos(syp.pi * ys) ** 2
    if which == "fluxdiv":
        exact = syp.diff(K * syp.diff(s, xs), xs) + syp.diff(K * syp.diff(s, ys), ys)
    else:  # the CH fourth-order operator div(K grad(Lap s))
        L = syp.diff(s, xs, 2) + syp.diff(s, ys, 2)
        exact = syp.diff(K * syp.diff(L, xs), xs) + syp.diff(K * syp.diff(L, ys), ys)
    f_s = syp.lambdify((xs, ys), s, "numpy")
    f_K = syp.lambdify((xs, ys), K, "numpy")
    f_e = syp.lambdify((xs, ys), exact, "numpy")
    X, Y = _grid(n, n)
    Xf = np.arange(n)[None, :] / n * np.ones((n, 1))
    Kx = f_K(Xf, Y)
    Yf = np.arange(n + 1)[:, None] / n * np.ones((1, n))
    Ky = f_K((np.arange(n)[None, :] + 0.5) / n, Yf)
    Ky[0] = Ky[-1] = 0.0                # wall faces: zero flux (the exact flux vanishes there too)
    sv = f_s(X, Y).ravel()
    L_K = asm.flux_div(n, n, Kx, Ky)
    got = L_K @ sv if which == "fluxdiv" else L_K @ (asm.lap(n, n) @ sv)
    return np.abs(got - f_e(X, Y).ravel()).max()


@pytest.mark.parametrize("which", ["fluxdiv", "ch4"])
def test_mms_second_order(which):
    errs = [_mms_error(n, which) for n in (16, 32, 64)]
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.2 < r1 < 4.8 and 3.2 < r2 < 4.8, errs


def test_ch_step_time_order_two():
    """CN + extrapolation: against the exact continuous-time decay of the linear
    mode (constant mobility via phi* = phi0), the error ratio is 4 per dt halving."""
    nx = ny = 16
    X, Y = _grid(nx, ny)
    e = np.cos(2 * np.pi * X) * np.cos(np.pi * Y)
    lam = -(4 * nx * nx) * np.sin(np.pi / nx) ** 2 - (4 * ny * ny) * np.sin(np.pi / (2 * ny)) ** 2
    phi0, d, T = 0.3, 1e-3, 0.2
    prm0 = Params(Lambda=1e-4, eps=0.0, rtol=1e-14)
    sigma = 0.5 * prm0.Gamma1 * prm0.Lambda * phi0 * lam ** 2 * 2   # d/dt amp = -G1 L phi0 lam^2 amp
    errs = []
    for dt in (2e-3, 1e-3, 5e-4):
        prm = prm0.with_(dt=dt)
        amp = d
        for _ in range(int(round(T / dt))):
            z = np.zeros((ny, nx))
            st = State(phi=phi0 + amp * e, phi_prev=phi0 + 3 * amp * e, c=np.ones((ny, nx)), u=z, v=z, p=z)
            A, b, phs = ch_system(st, prm)
            x, _ = bicgstab(A, b, phs.ravel(), 1 / A.diagonal(), 1e-14, 1000)
            amp = float(np.dot(x - phi0, e.ravel()) / np.dot(e.ravel(), e.ravel()))
        errs.append(abs(amp - d * math.exp(-sigma * T)))
    assert 3.5 < errs[0] / errs[1] < 4.5 and 3.5 < errs[1] / errs[2] < 4.5, errs


# ------------------------------------------------------------ invariants
def test_mass_conservation_and_projection_full_steps():
    """eps = 0: sum(phi) is conserved to round-off through the coupled step
    (conservative fluxes, zero-flux walls, v·n = 0); every step leaves a
    discretely divergence-free velocity (Eq. 21's purpose)."""
    n = 32
    st = initial_state(initial_fields(n, n, seed=5))
    prm = Params(eps=0.0)
    m0 = ex.mass(st.phi)
    for _ in range(4):
        prev = st
        st, info = step(st, prm)
        assert abs(ex.mass(st.phi) - m0) / m0 < 1e-12
        ref = np.abs(ex.divergence(*_ustar(prev, st, prm))).max()
        assert info.div_max <= 1e-8 * max(ref, 1e-300)


def _ustar(prev, new, prm):
    # reconstruct u* = v^{n+1} - beta grad p  (inverse of Eq. 21)
    bx, by = ex.pressure_faces(new.phi, prm.rho_n, prm.rho_s)
    return ex.correct(new.u, new.v, -new.p, bx, by)


def test_growth_adds_mass_exactly():
    """With v = 0 and production on, mass(phi^{n+1}) - mass(phi^n) = dt * mean(g_n(phi*, c^n))."""
    n = 16
    f = initial_fields(n, n, seed=2)
    st = initial_state(f)
    prm = Params(lid_u=0.0, Gamma1=0.0, rtol=1e-14)
    A, b, phs = ch_system(st, prm)
    x, _ = bicgstab(A, b, phs.ravel(), 1 / A.diagonal(), 1e-14, 100)
    g = ex.growth(phs, st.c, prm.eps, prm.mu, prm.Kc)
    assert (x.mean() - st.phi.mean()) == pytest.approx(prm.dt * g.mean(), rel=1e-9)


def test_free_energy_decays_pure_ch():
    """Spinodal decomposition with v = 0, no production: the discrete free
    energy (Eq. 16) is non-increasing after the start-up steps."""
    n = 32
    rng = np.random.default_rng(7)
    phi = 0.5 + 0.01 * (2 * rng.random((n, n)) - 1)
    prm = Params(Gamma1=1e-3, Gamma2=1.0, Lambda=1.0, eps=0.0, dt=5e-4, rtol=1e-10)
    z = np.zeros((n, n))
    st = State(phi=phi, phi_prev=phi.copy(), c=np.ones((n, n)), u=z, v=z, p=z)
    E = [ex.free_energy(st.phi, prm.Gamma1, prm.Gamma2)]
    for _ in range(150):
        A, b, phs = ch_system(st, prm)
        x, _ = bicgstab(A, b, phs.ravel(), 1 / A.diagonal(), prm.rtol, 5000)
        st = State(phi=x.reshape(n, n), phi_prev=st.phi, c=st.c, u=z, v=z, p=z)
        E.append(ex.free_energy(st.phi, prm.Gamma1, prm.Gamma2))
    E = np.array(E)
    assert np.all(np.diff(E[5:]) <= 1e-12 * E[0]), np.diff(E[5:]).max()
    assert E[-1] < 0.85 * E[0]               # real phase separation happened
    assert np.ptp(st.phi) > 0.8


# ---------------------------------------------------------- dense solves
@pytest.mark.parametrize("n", [8, 16])
def test_krylov_matches_dense_direct_solve(n):
    st = initial_state(initial_fields(n, n, seed=11))
    prm = Params(Lambda=1e-3)            # make the CH system far from I/dt
    A, b, phs = ch_system(st, prm)
    ref = np.linalg.solve(A.toarray(), b)
    d = 1 / A.diagonal()
    for solver in (lambda: bicgstab(A, b, phs.ravel(), d, 1e-12, 5000),
                   lambda: gmres(A, b, phs.ravel(), d, 1e-12, 5000, restart=10)):
        x, _ = solver()
        assert _rel(x, ref) < 1e-9
    st2, _ = step(st, Params())
    An, bn = nutrient_system(st, st2.phi, prm)
    x, _ = cg(An, bn, st.c.ravel(), 1 / An.diagonal(), 1e-12, 5000)
    assert _rel(x, np.linalg.solve(An.toarray(), bn)) < 1e-9
    (Au, bu), (Av, bv) = momentum_systems(st, phs, prm)
    for M, rhs in ((Au, bu), (Av, bv)):
        x, _ = cg(M, rhs, np.zeros_like(rhs), 1 / M.diagonal(), 1e-12, 5000)
        assert _rel(x, np.linalg.solve(M.toarray(), rhs)) < 1e-9
    bx, by = ex.pressure_faces(st2.phi, 1.0, 1.0)
    Ap = asm.poisson_matrix(n, n, bx, by).toarray()
    rhs = np.random.default_rng(0).standard_normal(n * n)
    rhs -= rhs.mean()
    ref = np.linalg.lstsq(Ap, rhs, rcond=None)[0]
    ref -= ref.mean()
    x, _ = cg(sp.csr_matrix(Ap), rhs, np.zeros(n * n), 1 / np.diag(Ap), 1e-12, 5000, nullspace=True)
    assert _rel(x, ref) < 1e-8
    assert abs(x.mean()) <= 1e-12 * np.abs(x).max()


def test_nonsymmetric_ch_operator():
    """The CH system is nonsymmetric (why BiCGStab/GMRES), the others are symmetric."""
    n = 8
    st = initial_state(initial_fields(n, n, seed=1))
    A, _, _ = ch_system(st, Params(Lambda=1.0))
    assert abs(A - A.T).max() > 1e-6 * abs(A).max()
    (Au, _), (Av, _) = momentum_systems(st, ex.phi_star(st.phi, st.phi_prev), Params())
    assert abs(Au - Au.T).max() <= 1e-12 * abs(Au).max()
    assert abs(Av - Av.T).max() <= 1e-12 * abs(Av).max()


def test_inputs_decomposition_invisible():
    full = initial_fields(40, 30, seed=9)
    part = initial_fields(40, 30, seed=9, rows=(7, 19))
    assert np.array_equal(full["phi"][7:19], part["phi"])
    phi = full["phi"]
    assert phi.min() >= 0.0 and phi.max() <= 0.301
    X, Y = _grid(40, 30)
    assert np.all(phi[Y < 0.2] > 0.29)


def test_stratified_phase_stress_is_balanced_by_pressure():
    """phi = phi(y) (flat interface), fluid at rest, lid off: the phase stress
    R = -G1 div(grad phi grad phi) is a pure y-gradient, so the projected
    velocity stays zero and the pressure alone balances it.  The expected p is
    an independent 1D reduction (tridiagonal dense solve for v*, then the
    cumulative sum of Eq. 21 with v^{n+1} = 0)."""
    nx, ny = 6, 24
    y = (np.arange(ny) + 0.5) / ny
    prof = 0.3 * 0.5 * (1 + np.tanh((0.5 - y) / 0.08))
    phi = np.repeat(prof[:, None], nx, axis=1)
    prm = Params(lid_u=0.0, eps=0.0, A=0.0, Re_n=1e-2, Re_s=1.0, dt=1e-3, rtol=1e-14)
    z = np.zeros((ny, nx))
    st = State(phi=phi, phi_prev=phi.copy(), c=np.ones((ny, nx)), u=z, v=z, p=z)
    new, _ = step(st, prm)
    assert np.abs(new.u).max() < 1e-10 and np.abs(new.v).max() < 1e-10
    # 1D reduction
    h = 1.0 / ny
    gy = np.empty(ny)
    gy[1:-1] = (prof[2:] - prof[:-2]) / (2 * h)
    gy[0] = (prof[1] - prof[0]) / (2 * h)       # mirror ghost
    gy[-1] = (prof[-1] - prof[-2]) / (2 * h)
    Tyy = gy ** 2
    Ry = -prm.Gamma1 * (Tyy[1:] - Tyy[:-1]) / h           # faces j = 1..ny-1
    fphi = 0.5 * (prof[1:] + prof[:-1])
    nu = fphi / prm.Re_n + (1 - fphi) / prm.Re_s
    a = 1 / (nu * prm.dt)
    m = ny - 1
    M = np.diag(a + 1 / h ** 2) - np.diag(np.full(m - 1, 0.5 / h ** 2), 1) - np.diag(np.full(m - 1, 0.5 / h ** 2), -1)
    vstar = np.linalg.solve(M, Ry / nu)
    p = np.concatenate([[0.0], np.cumsum(-vstar * h)])    # beta = 1 (rho_n = rho_s)
    p -= p.mean()
    assert np.abs(p).max() > 1e-6
    assert _rel(new.p[:, 0], p) < 1e-9
    assert np.abs(new.p - new.p[:, :1]).max() < 1e-12
