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
    uu = rng.standard_normal((ny, nx))
    vv = rng.standard_normal((ny, nx))
    vv[0] = 0.0
    A = asm.ch_matrix(nx, ny, prm.dt, prm.Gamma1, Mx, My, 0.7, 0.4, uu, vv)
    assert _rel(A @ x.ravel(), brute.ch_apply(phis, x, prm.dt, prm.Gamma1, prm.Lambda,
                                              0.7, 0.4, uu, vv)) < 1e-13
    bx, by = ex.pressure_faces(phis, 2.0, 1.0)
    assert _rel(asm.poisson_matrix(nx, ny, bx, by) @ x.ravel(),
                brute.poisson_apply(phis, x, 2.0, 1.0)) < 1e-13
    a = 1.0 + rng.random((ny, nx))
    eta = 0.5 + rng.random((ny, nx))
    K = ex.node_fluxes(eta)
    for th in (1.0, 0.5):
        assert _rel(asm.u_matrix(nx, ny, a, K, th) @ x.ravel(), brute.u_apply(a, eta, x, th)) < 1e-13
        xv = x.copy()
        xv[0] = 0.0
        assert _rel(asm.v_matrix(nx, ny, a, K, th) @ xv.ravel(),
                    brute.v_apply(a, eta, xv, th)) < 1e-13
    # the explicit parts of the momentum right-hand side
    ue = rng.standard_normal((ny, nx))
    ve = rng.standard_normal((ny, nx))
    ve[0] = 0.0
    phv = rng.uniform(-0.1, 1.1, (ny, nx))   # exercises the volume-fraction clip (R24)
    tx, ty = brute.visc_transpose(ue, ve, phv, 0.3, 2.0)
    Tx, Ty = ex.visc_transpose(ue, ve, phv, 0.3, 2.0)
    assert _rel(Tx, tx) < 1e-13 and _rel(Ty, ty) < 1e-13
    lid = 0.7
    assert _rel(ex.visc_u_inhom(ue, eta, 0.0), -brute.u_apply(np.zeros_like(a), eta, ue)) < 1e-13
    assert _rel(ex.visc_v(ve, eta)[1:], -brute.v_apply(np.zeros_like(a), eta, ve)[1:]) < 1e-13
    lidpart = ex.visc_u_inhom(ue, eta, lid) - ex.visc_u_inhom(ue, eta, 0.0)
    assert np.abs(lidpart[:-1]).max() < 1e-9
    assert _rel(lidpart[-1], 2 * lid * eta[-1] * ny * ny) < 1e-13
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
    prm = Params(Lambda=0.1, eps=0.0, rtol=1e-14, startup_be=0)
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
    convection and R (incl. its viscous part) vanish, D u* = 0 so p = 0, and
    the full step multiplies the mode by (a + (1-th) lam)/(a - th lam),
    a = rho/(eta dt): a/(a - lam) for the implicit viscous term of Eq. 19
    (th = 1, R7), (a + lam/2)/(a - lam/2) for Crank-Nicolson."""
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
    for th in (1.0, 0.5):
        st = State(phi=np.full((ny, nx), phi0), phi_prev=np.full((ny, nx), phi0),
                   c=np.ones((ny, nx)), u=d * e, v=z.copy(), p=z.copy())
        new, info = step(st, prm.with_(theta_visc=th))
        assert _rel(new.u, d * e * (a + (1 - th) * lam) / (a - th * lam)) < 1e-12
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
    prm0 = Params(Lambda=1e-4, eps=0.0, rtol=1e-14, startup_be=0)
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
        st = State(phi=x.reshape(n, n), phi_prev=st.phi, c=st.c, u=z, v=z, p=z, n=st.n + 1)
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
    # implicit viscous operator rho/dt - d/dy(eta d/dy) on the v points j = 1..ny-1
    # (v = 0 on both walls), eta at the v points from the face mean of phi
    # (row 0: the wall, phi[0]), face coefficients = mean of the two (R6)
    fphi = np.concatenate([[prof[0]], 0.5 * (prof[1:] + prof[:-1])])
    eta = fphi / prm.Re_n + (1 - fphi) / prm.Re_s
    etap = np.concatenate([eta, [eta[-1]]])           # mirror ghost above the top point
    KS = 0.5 * (eta[:-1] + eta[1:])                   # between points j-1 and j, j = 1..ny-1
    KN = 0.5 * (eta[1:] + etap[2:])                   # between j and j+1
    M = (np.diag(1 / prm.dt + (KS + KN) / h ** 2) - np.diag(KN[:-1] / h ** 2, 1)
         - np.diag(KS[1:] / h ** 2, -1))
    vstar = np.linalg.solve(M, Ry)
    p = np.concatenate([[0.0], np.cumsum(-vstar * h)])    # beta = 1 (rho_n = rho_s)
    p -= p.mean()
    assert np.abs(p).max() > 1e-6
    assert _rel(new.p[:, 0], p) < 1e-9
    assert np.abs(new.p - new.p[:, :1]).max() < 1e-12


# ------------------------------------------------- implicit advection (R12)
def _streamfunction_velocity(nx, ny, seed):
    """Discretely divergence-free MAC velocity from a random corner stream
    function psi with psi = 0 on both walls: u = d psi/dy on x-faces,
    v = -d psi/dx on y-faces (so D_h(u, v) = 0 exactly and v = 0 on the walls)."""
    rng = np.random.default_rng(seed)
    psi = rng.standard_normal((ny + 1, nx))
    psi[0] = psi[-1] = 0.0
    u = (psi[1:] - psi[:-1]) * ny
    v = -(np.roll(psi, -1, axis=1) - psi)[:ny] * nx
    return u, v


def test_advection_matrix_structure():
    """Central conservative fluxes: A + A^T = diag(D_h v) (skew-symmetric for a
    discretely divergence-free v), A 1 = D_h v, and the column sums vanish
    (telescoping fluxes, zero wall flux)."""
    nx, ny = 7, 6
    rng = np.random.default_rng(4)
    u = rng.standard_normal((ny, nx))
    v = rng.standard_normal((ny, nx))
    v[0] = 0.0
    A = asm.advection_matrix(nx, ny, u, v)
    div = ex.divergence(u, v).ravel()
    assert abs(A + A.T - sp.diags(div)).max() < 1e-12 * nx
    assert np.abs(A @ np.ones(nx * ny) - div).max() < 1e-12 * nx
    assert np.abs(np.ones(nx * ny) @ A).max() < 1e-12 * nx
    us, vs = _streamfunction_velocity(nx, ny, 1)
    assert np.abs(ex.divergence(us, vs)).max() < 1e-12 * nx * ny
    B = asm.advection_matrix(nx, ny, us, vs)
    assert abs(B + B.T).max() < 1e-11 * nx * ny


@pytest.mark.parametrize("startup", [0, 1])
def test_ch_advection_translation_closed_form(startup):
    """Pure translation u = U, v = 0, no CH flux (Lambda = 0), no production:
    the x-mode cos(2 pi k x) is an eigenvector of the central advection with
    eigenvalue i U sin(2 pi k h)/h, so one CH step multiplies its complex
    amplitude by (1 - (1-ta) dt i s)/(1 + ta dt i s), ta = 1/2 (CN, R12) or 1
    in a backward-Euler start-up step (R23)."""
    nx, ny = 16, 6
    X, Y = _grid(nx, ny)
    k, U, d, phi0 = 3, 2.0, 1e-2, 0.3
    prm = Params(Lambda=0.0, eps=0.0, dt=0.02, startup_be=startup)
    z = np.zeros((ny, nx))
    phi = phi0 + d * np.cos(2 * np.pi * k * X)
    st = State(phi=phi, phi_prev=phi.copy(), c=np.ones((ny, nx)), u=np.full((ny, nx), U),
               v=z, p=z)
    A, b, phs = ch_system(st, prm)
    x, _ = bicgstab(A, b, phs.ravel(), 1 / A.diagonal(), 1e-14, 1000)
    ta = 1.0 if startup else 0.5
    s = U * math.sin(2 * np.pi * k / nx) * nx
    g = (1 - (1 - ta) * prm.dt * 1j * s) / (1 + ta * prm.dt * 1j * s)
    assert abs(g) < 1 if startup else abs(abs(g) - 1) < 1e-15
    exact = phi0 + d * np.real(g * np.exp(2j * np.pi * k * X))
    assert _rel(x, exact.ravel()) < 1e-12


def test_cn_advection_conserves_mass_and_l2():
    """Crank-Nicolson central advection with a discretely divergence-free v is
    an isometry (Cayley transform of a skew-symmetric operator): ||phi||_2 and
    sum(phi) are conserved to solver precision, at a Courant number > 1."""
    nx, ny = 24, 20
    u, v = _streamfunction_velocity(nx, ny, 2)
    u, v = u / 50, v / 50
    rng = np.random.default_rng(5)
    phi = rng.random((ny, nx))
    prm = Params(Lambda=0.0, eps=0.0, dt=0.05, startup_be=0)
    cfl = prm.dt * max(np.abs(u).max() * nx, np.abs(v).max() * ny)
    assert cfl > 1.0
    st = State(phi=phi, phi_prev=phi.copy(), c=np.ones((ny, nx)), u=u, v=v, p=np.zeros((ny, nx)))
    A, b, phs = ch_system(st, prm)
    x, _ = bicgstab(A, b, phs.ravel(), 1 / A.diagonal(), 1e-13, 5000)
    assert abs(np.linalg.norm(x) - np.linalg.norm(phi)) < 1e-12 * np.linalg.norm(phi)
    assert abs(x.sum() - phi.sum()) < 1e-12 * phi.sum()
    assert _rel(x, phi.ravel()) > 1e-2          # it did move


def test_ch_startup_step_is_backward_euler():
    """With startup_be = 1 the first CH step takes theta = 1 on the Gamma1 term:
    the eigenmode factor is (1/dt)/(1/dt + G1 L phi0 lam^2) (R23); the second
    step is Crank-Nicolson again."""
    nx, ny = 16, 16
    X, Y = _grid(nx, ny)
    e = np.cos(2 * np.pi * X) * np.cos(np.pi * 2 * Y)
    lam = -(4 * nx * nx) * np.sin(np.pi / nx) ** 2 - (4 * ny * ny) * np.sin(np.pi / ny) ** 2
    phi0, d = 0.3, 1e-3
    prm = Params(Lambda=0.1, eps=0.0, startup_be=1)
    z = np.zeros((ny, nx))
    q = prm.Gamma1 * prm.Lambda * phi0 * lam ** 2
    for n, g in ((0, (1 / prm.dt) / (1 / prm.dt + q)),
                 (1, (1 / prm.dt - q / 2) / (1 / prm.dt + q / 2))):
        st = State(phi=phi0 + d * e, phi_prev=phi0 + 3 * d * e, c=np.ones((ny, nx)), u=z, v=z,
                   p=z, n=n)
        A, b, phs = ch_system(st, prm)
        x, _ = bicgstab(A, b, phs.ravel(), 1.0 / A.diagonal(), 1e-14, 1000)
        assert _rel(x - phi0, d * g * e.ravel()) < 1e-10


# ------------------------------------- momentum pieces against analytic fields
def _u_points(n):
    x = np.arange(n)[None, :] / n * np.ones((n, 1))
    y = (np.arange(n)[:, None] + 0.5) / n * np.ones((1, n))
    return x, y


def _v_points(n):
    x = (np.arange(n)[None, :] + 0.5) / n * np.ones((n, 1))
    y = np.arange(n)[:, None] / n * np.ones((1, n))
    return x, y


def _order(errs):
    return [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]


def test_viscous_flux_form_second_order():
    """div_h(eta grad_h u) on the u points (odd walls) against the analytic
    div(eta grad s), s = cos(2 pi x) sin(pi y) (zero on the walls), eta =
    1 + sin(2 pi x) cos(pi y)^2 / 2 (even about the walls): error ratio 4."""
    errs = []
    for n in (16, 32, 64):
        X, Y = _u_points(n)
        s = np.cos(2 * np.pi * X) * np.sin(np.pi * Y)
        eta = 1 + 0.5 * np.sin(2 * np.pi * X) * np.cos(np.pi * Y) ** 2
        sx = -2 * np.pi * np.sin(2 * np.pi * X) * np.sin(np.pi * Y)
        sy = np.pi * np.cos(2 * np.pi * X) * np.cos(np.pi * Y)
        ex_ = np.pi * np.cos(2 * np.pi * X) * np.cos(np.pi * Y) ** 2
        ey_ = -0.5 * np.sin(2 * np.pi * X) * 2 * np.cos(np.pi * Y) * np.sin(np.pi * Y) * np.pi
        sxx = -4 * np.pi ** 2 * s
        syy = -np.pi ** 2 * s
        exact = ex_ * sx + eta * sxx + ey_ * sy + eta * syy
        got = ex.visc_u_inhom(s, eta, 0.0)
        errs.append(np.abs(got - exact).max())
    r = _order(errs)
    assert all(3.3 < q < 4.7 for q in r), errs


def test_viscous_transpose_analytic_and_identity():
    """R's viscous part div(eta (grad v)^T): (a) shear u = sin(pi y), v = 0 under
    eta = eta(x): T_x = 0 and T_y = eta'(x) u'(y) at second order; (b) constant eta
    and a discretely divergence-free v: T = eta grad(div v) = 0 to round-off."""
    Re_n, Re_s = 0.5, 2.0                       # eta(phi) = phi/Re_n + (1-phi)/Re_s
    errs = []
    for n in (16, 32, 64):
        xc = (np.arange(n) + 0.5) / n
        phis = np.repeat((0.5 + 0.4 * np.sin(2 * np.pi * xc))[None, :], n, axis=0)
        Xu, Yu = _u_points(n)
        u = np.sin(np.pi * Yu)
        Tx, Ty = ex.visc_transpose(u, np.zeros((n, n)), phis, Re_n, Re_s)
        assert np.abs(Tx).max() < 1e-9
        Xv, Yv = _v_points(n)                   # T_y lives on the v points (j >= 1)
        deta = (1 / Re_n - 1 / Re_s) * 0.4 * 2 * np.pi * np.cos(2 * np.pi * Xv)
        exact = deta * np.pi * np.cos(np.pi * Yv)
        errs.append(np.abs(Ty[1:] - exact[1:]).max())
    assert all(3.3 < q < 4.7 for q in _order(errs)), errs
    nx, ny = 12, 10
    us, vs = _streamfunction_velocity(nx, ny, 3)
    Tx, Ty = ex.visc_transpose(us, vs, np.full((ny, nx), 0.3), Re_n, Re_s)
    assert np.abs(Tx).max() < 1e-9 * np.abs(us).max() * nx * nx
    assert np.abs(Ty).max() < 1e-9 * np.abs(us).max() * nx * nx


def test_convective_terms_second_order():
    """(v·∇)u on the u points and (v·∇)v on the v points against analytic
    fields: u = U + sin(2 pi x) sin(pi y) ... evaluated where each lives."""
    eu, ev = [], []
    for n in (16, 32, 64):
        Xu, Yu = _u_points(n)
        Xv, Yv = _v_points(n)
        A, B = 0.7, 0.4
        # u = A sin(2 pi x) sin(pi y) (zero on the walls, lid 0);  v = B sin(2 pi x) sin(pi y)
        uf = lambda x, y: A * np.sin(2 * np.pi * x) * np.sin(np.pi * y)
        vf = lambda x, y: B * np.sin(2 * np.pi * x) * np.sin(np.pi * y)
        u, v = uf(Xu, Yu), vf(Xv, Yv)
        v[0] = 0.0
        ux = lambda x, y: A * 2 * np.pi * np.cos(2 * np.pi * x) * np.sin(np.pi * y)
        uy = lambda x, y: A * np.pi * np.sin(2 * np.pi * x) * np.cos(np.pi * y)
        vx = lambda x, y: B * 2 * np.pi * np.cos(2 * np.pi * x) * np.sin(np.pi * y)
        vy = lambda x, y: B * np.pi * np.sin(2 * np.pi * x) * np.cos(np.pi * y)
        cu = uf(Xu, Yu) * ux(Xu, Yu) + vf(Xu, Yu) * uy(Xu, Yu)
        cv = uf(Xv, Yv) * vx(Xv, Yv) + vf(Xv, Yv) * vy(Xv, Yv)
        eu.append(np.abs(ex.convective_u(u, v, 0.0) - cu).max())
        ev.append(np.abs((ex.convective_v(u, v) - cv)[1:]).max())
    assert all(3.3 < q < 4.7 for q in _order(eu)), eu
    assert all(3.3 < q < 4.7 for q in _order(ev)), ev


def test_phase_stress_second_order():
    """R = -G1 div(grad phi (x) grad phi) for phi = cos(2 pi x) cos(pi y) against
    the analytic divergence (all of T_xx, T_yy, T_xy enter), error ratio 4."""
    G1 = 1.3
    ex_, ey_ = [], []
    for n in (16, 32, 64):
        X, Y = _grid(n, n)
        phi = np.cos(2 * np.pi * X) * np.cos(np.pi * Y)
        p = lambda x, y: np.cos(2 * np.pi * x) * np.cos(np.pi * y)
        px = lambda x, y: -2 * np.pi * np.sin(2 * np.pi * x) * np.cos(np.pi * y)
        py = lambda x, y: -np.pi * np.cos(2 * np.pi * x) * np.sin(np.pi * y)
        pxx = lambda x, y: -4 * np.pi ** 2 * p(x, y)
        pyy = lambda x, y: -np.pi ** 2 * p(x, y)
        pxy = lambda x, y: 2 * np.pi ** 2 * np.sin(2 * np.pi * x) * np.sin(np.pi * y)
        # div(grad phi grad phi) = (lap phi) grad phi + grad(|grad phi|^2)/2
        rx = lambda x, y: -G1 * ((pxx(x, y) + pyy(x, y)) * px(x, y)
                                 + px(x, y) * pxx(x, y) + py(x, y) * pxy(x, y))
        ry = lambda x, y: -G1 * ((pxx(x, y) + pyy(x, y)) * py(x, y)
                                 + px(x, y) * pxy(x, y) + py(x, y) * pyy(x, y))
        Rx, Ry = ex.phase_stress(phi, G1)
        Xu, Yu = _u_points(n)
        Xv, Yv = _v_points(n)
        ex_.append(np.abs(Rx - rx(Xu, Yu)).max())
        ey_.append(np.abs((Ry - ry(Xv, Yv))[1:]).max())
    assert all(3.3 < q < 4.7 for q in _order(ex_)), ex_
    assert all(3.3 < q < 4.7 for q in _order(ey_)), ey_


def test_growth_uniform_state_closed_form():
    """Uniform phi0, c0, v = 0: one CH step adds exactly dt eps mu phi0 c0/(K_c + c0)
    (Eq. 5 by hand) -- and nothing for phi0 < 0 (volume fraction, R24)."""
    n = 8
    z = np.zeros((n, n))
    prm = Params(dt=0.01, eps=1.0, mu=0.14, Kc=0.15, lid_u=0.0, rtol=1e-14)
    for phi0, c0, gain in ((0.3, 0.8, 0.01 * 0.14 * 0.3 * 0.8 / 0.95), (-0.01, 0.8, 0.0)):
        st = State(phi=np.full((n, n), phi0), phi_prev=np.full((n, n), phi0),
                   c=np.full((n, n), c0), u=z, v=z, p=z)
        A, b, phs = ch_system(st, prm)
        x, _ = bicgstab(A, b, phs.ravel(), 1 / A.diagonal(), 1e-14, 100)
        assert np.abs(x - (phi0 + gain)).max() < 1e-15 + 1e-13 * abs(phi0)


@pytest.mark.parametrize("phi0", [0.3, 0.7, 0.05])
def test_fprime_linear_growth_rate(phi0):
    """Gamma1 = 0, v = 0, no production, phi^n = phi^{n-1} = phi0 + d e (e a
    Laplacian eigenmode with eigenvalue lam): one CH step multiplies the mode by
    1 + dt Lambda phi0 F''(phi0) lam + O(d), with F''(phi) = 2 Gamma2 (1 - 6 phi
    + 6 phi^2) the second derivative of Gamma2 phi^2 (1 - phi)^2 (Eq. 16 energy,
    PAPER.md:113).  Two amplitudes extrapolate the O(d) term away."""
    nx, ny = 16, 12
    X, Y = _grid(nx, ny)
    e = np.cos(2 * np.pi * X) * np.cos(np.pi * Y)
    lam = -(4 * nx * nx) * np.sin(np.pi / nx) ** 2 - (4 * ny * ny) * np.sin(np.pi / (2 * ny)) ** 2
    prm = Params(Gamma1=0.0, Gamma2=2.0, Lambda=1.0, eps=0.0, dt=0.01, lid_u=0.0)
    z = np.zeros((ny, nx))
    amps = []
    for d in (1e-4, 2e-4):
        phi = phi0 + d * e
        st = State(phi=phi, phi_prev=phi.copy(), c=np.ones((ny, nx)), u=z, v=z, p=z)
        A, b, phs = ch_system(st, prm)
        x = b * prm.dt                                   # A = I/dt exactly (Gamma1 = 0, v = 0)
        amps.append(float(np.dot(x - phi0, e.ravel()) / np.dot(e.ravel(), e.ravel())) / d)
    g = 2 * amps[0] - amps[1]                            # Richardson in d
    F2 = 2 * prm.Gamma2 * (1 - 6 * phi0 + 6 * phi0 ** 2)
    expect = 1 + prm.dt * prm.Lambda * phi0 * F2 * lam
    assert abs(expect - 1) > 1e-3                        # the pin is non-trivial
    assert abs(g - expect) < 1e-6 * abs(expect - 1)
