"""One semi-implicit time step of the biofilm model.  Test infrastructure only.

Splitting order (R1): Cahn-Hilliard -> nutrient -> momentum
(Chorin projection: intermediate velocity, pressure Poisson, correction).
PAPER.md §4 (lines 117-151) and Eq. 16 (lines 108-114).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import assemble as asm
from . import explicit as ex
from .krylov import bicgstab, cg, gmres
from .params import Params


@dataclass
class State:
    phi: np.ndarray        # phi_n^n       (ny, nx) cell centres
    phi_prev: np.ndarray   # phi_n^{n-1}
    c: np.ndarray          # nutrient c^n  cell centres
    u: np.ndarray          # x-velocity on x-faces
    v: np.ndarray          # y-velocity on y-faces (row 0 = bottom wall = 0)
    p: np.ndarray          # pressure (paper's Eq. 20 variable, Δt absorbed; R15)
    n: int = 0
    us: np.ndarray | None = None   # u* of the previous step: initial guess of the
    vs: np.ndarray | None = None   # next momentum solves (R25); None -> u, v

    def copy(self) -> "State":
        return State(self.phi.copy(), self.phi_prev.copy(), self.c.copy(),
                     self.u.copy(), self.v.copy(), self.p.copy(), self.n,
                     None if self.us is None else self.us.copy(),
                     None if self.vs is None else self.vs.copy())

    def guess_uv(self):
        """Initial guesses of the momentum solves (R25): the previous step's
        intermediate velocity (u*, v*), or (u, v) when there is none (the
        first step after an initial condition is set)."""
        return (self.u if self.us is None else self.us,
                self.v if self.vs is None else self.vs)


@dataclass
class StepInfo:
    iters: dict = field(default_factory=dict)
    div_max: float = 0.0


def initial_state(fields: dict) -> State:
    """phi^{-1} := phi^0 (first step extrapolates to phi* = phi^0, R5)."""
    return State(phi=fields["phi"].copy(), phi_prev=fields["phi"].copy(),
                 c=fields["c"].copy(), u=fields["u"].copy(),
                 v=fields["v"].copy(), p=fields["p"].copy())


def _solve_ch(A, b, x0, dinv, prm: Params):
    if prm.ch_solver == "gmres":
        return gmres(A, b, x0, dinv, prm.rtol, prm.maxit, prm.gmres_restart)
    return bicgstab(A, b, x0, dinv, prm.rtol, prm.maxit)


def ch_thetas(st: State, prm: Params):
    """Implicit weights of the step at time index st.n: the CN weights, or 1
    during the backward-Euler start-up steps (R23)."""
    if st.n < prm.startup_be:
        return 1.0, 1.0
    return prm.theta_ch, prm.theta_adv


def ch_system(st: State, prm: Params):
    """Linear system of the CH step (Eq. 16 4th line, Eq. 4-5; R5, R12):
      [I/dt + th G1 L_{M*} Δ_h + ta Adv(.; v^n)] phi^{n+1}
        = phi^n/dt + L_{M*}( F'(phi*) - (1-th) G1 Δ_h phi^n )
          - (1-ta) Adv(phi^n; v^n) + g_n(phi*, c^n)
    with th = theta_ch, ta = theta_adv (1/2: Crank-Nicolson).  Returns (A, b, phi*)."""
    ny, nx = st.phi.shape
    th, ta = ch_thetas(st, prm)
    phs = ex.phi_star(st.phi, st.phi_prev)
    Mx, My = ex.mobility_faces(phs, prm.Lambda)
    L_M = asm.flux_div(nx, ny, Mx, My)
    Lap = asm.lap(nx, ny, "mirror")
    A = asm.ch_matrix(nx, ny, prm.dt, prm.Gamma1, Mx, My, th, ta, st.u, st.v)
    mu_e = ex.fprime(phs, prm.Gamma2).ravel() - (1.0 - th) * prm.Gamma1 * (Lap @ st.phi.ravel())
    b = (st.phi.ravel() / prm.dt + L_M @ mu_e
         - (1.0 - ta) * ex.advection(st.phi, st.u, st.v).ravel()
         + ex.growth(phs, st.c, prm.eps, prm.mu, prm.Kc).ravel())
    return A, b, phs


def nutrient_system(st: State, phi1: np.ndarray, prm: Params):
    """Nutrient step (Eq. 16 3rd line, Eq. 7; R11), Crank-Nicolson diffusion and
    consumption, explicit advection of phi_s c at level n:
      [diag(phi_s^{n+1}/dt + A/2 phi_n^{1/2}) - 1/2 L_K] c^{n+1}
        = phi_s^n c^n/dt - div_h(phi_s^n c^n v^n) + 1/2 L_K c^n - A/2 phi_n^{1/2} c^n,
    K = D_s phi_s^{1/2} on faces; phi_n^{1/2} = clip((phi^n + phi^{n+1})/2),
    phi_s = 1 - clip(phi) (volume fractions, R24)."""
    ny, nx = st.phi.shape
    vf = ex.volume_fraction
    ph = vf(0.5 * (st.phi + phi1))
    sh = 1.0 - ph
    s1 = 1.0 - vf(phi1)
    s0 = 1.0 - vf(st.phi)
    Kx = prm.Ds * 0.5 * (np.roll(sh, 1, axis=1) + sh)
    Ky = np.zeros((ny + 1, nx))
    Ky[1:ny] = prm.Ds * 0.5 * (sh[:-1] + sh[1:])
    a_c = s1 / prm.dt + 0.5 * prm.A * ph
    A = asm.nutrient_matrix(nx, ny, a_c, Kx, Ky)
    L_K = asm.flux_div(nx, ny, Kx, Ky)
    w = s0 * st.c
    b = (w.ravel() / prm.dt - ex.advection(w, st.u, st.v).ravel()
         + 0.5 * (L_K @ st.c.ravel()) - (0.5 * prm.A * ph * st.c).ravel())
    return A, b


def momentum_systems(st: State, phs: np.ndarray, prm: Params):
    """Intermediate velocity (Eq. 18-19 with R restored, R6-R7), per component,
    SPD, th = theta_visc (1: the viscous term at u^{n+1}, the BVP of Eq. 19 as
    printed), eta = 1/Re_a and rho at phi* (R6, R24):
      [rho/dt - th div(eta grad)] u* = rho u^n/dt + (1-th) div(eta grad u^n) + th lid
                                       - rho (v^n·∇)u^n + R_x,
      R = -Gamma1 div(grad phi* grad phi*) + div(eta (grad v^n)^T)   (Eq. 17)."""
    ny, nx = st.phi.shape
    hy = 1.0 / ny
    th = prm.theta_visc
    Rx, Ry = ex.phase_stress(phs, prm.Gamma1)
    Tx, Ty = ex.visc_transpose(st.u, st.v, phs, prm.Re_n, prm.Re_s)
    rho_u = ex.density(ex.face_phi_u(phs), prm.rho_n, prm.rho_s)
    rho_v = ex.density(ex.face_phi_v(phs), prm.rho_n, prm.rho_s)
    eta_u = ex.viscosity_u(phs, prm.Re_n, prm.Re_s)
    eta_v = ex.viscosity_v(phs, prm.Re_n, prm.Re_s)
    a_u = rho_u / prm.dt
    a_v = rho_v / prm.dt
    Cu = ex.convective_u(st.u, st.v, prm.lid_u)
    Cv = ex.convective_v(st.u, st.v)
    bu = (a_u * st.u + (1.0 - th) * ex.visc_u_inhom(st.u, eta_u, prm.lid_u)
          - rho_u * Cu + Rx + Tx)
    Ku = ex.node_fluxes(eta_u)
    bu[-1] += th * Ku[3][-1] * 2.0 * prm.lid_u / hy ** 2   # implicit part of the lid ghost (R3)
    bv = a_v * st.v + (1.0 - th) * ex.visc_v(st.v, eta_v) - rho_v * Cv + Ry + Ty
    bv[0] = 0.0
    Au = asm.u_matrix(nx, ny, a_u, Ku, th)
    Av = asm.v_matrix(nx, ny, a_v, ex.node_fluxes(eta_v), th)
    return (Au, bu.ravel()), (Av, bv.ravel())


def step(st: State, prm: Params) -> tuple[State, StepInfo]:
    ny, nx = st.phi.shape
    info = StepInfo()
    # 1. Cahn-Hilliard (phi^{n+1}); initial guess phi* (R13)
    A, b, phs = ch_system(st, prm)
    dinv = 1.0 / A.diagonal()
    phi1, info.iters["ch"] = _solve_ch(A, b, phs.ravel(), dinv, prm)
    phi1 = phi1.reshape(ny, nx)
    # 2. nutrient (c^{n+1}); guess c^n
    A, b = nutrient_system(st, phi1, prm)
    c1, info.iters["nutrient"] = cg(A, b, st.c.ravel(), 1.0 / A.diagonal(), prm.rtol, prm.maxit)
    c1 = c1.reshape(ny, nx)
    # 3. intermediate velocity (u*, v*); guesses u*, v* of the previous step (R25)
    (Au, bu), (Av, bv) = momentum_systems(st, phs, prm)
    gu, gv = st.guess_uv()
    us, info.iters["u"] = cg(Au, bu, gu.ravel(), 1.0 / Au.diagonal(), prm.rtol, prm.maxit)
    vs, info.iters["v"] = cg(Av, bv, gv.ravel(), 1.0 / Av.diagonal(), prm.rtol, prm.maxit)
    us, vs = us.reshape(ny, nx), vs.reshape(ny, nx)
    # 4. pressure Poisson (Eq. 20) with constant null space removed; guess p^n
    bx, by = ex.pressure_faces(phi1, prm.rho_n, prm.rho_s)
    Ap = asm.poisson_matrix(nx, ny, bx, by)
    bp = ex.divergence(us, vs).ravel()
    p1, info.iters["p"] = cg(Ap, bp, st.p.ravel(), 1.0 / Ap.diagonal(), prm.rtol, prm.maxit,
                             nullspace=True)
    p1 = p1.reshape(ny, nx)
    # 5. projection (Eq. 21)
    u1, v1 = ex.correct(us, vs, p1, bx, by)
    info.div_max = float(np.abs(ex.divergence(u1, v1)).max())
    new = State(phi=phi1, phi_prev=st.phi.copy(), c=c1, u=u1, v=v1, p=p1, n=st.n + 1,
                us=us, vs=vs)
    return new, info


def run(st: State, prm: Params, steps: int, callback=None) -> State:
    for _ in range(steps):
        st, info = step(st, prm)
        if callback is not None:
            callback(st, info)
    return st

