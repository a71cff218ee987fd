"""Model parameters (§3 Eq. 15, §5).  Test infrastructure only.

Dimensionless values default to the paper's §5 block:
  Re_s = 9.98e-4, Re_n = 2.33e-9, Lambda = 1e-10, Gamma1 = 33.467,
  Gamma2 = 1.25e6, D_s = 2.3, mu = 0.14, K_c = 0.15, A = 100.
epsilon (Eq. 5, "a scaling constant", no value printed) defaults to 1 [R8].
rho_n/rho_0 = rho_s/rho_0 = 1 (Table 1 lists both densities as 1e3) [R9].
lid_u: top-wall tangential velocity; BASELINE.json reads "u = y at the top
wall", i.e. u(x, 1) = 1 [R10]; the paper's §5.1 run used 0.1 (Eq. 22).

Time discretisation (implicit weights, R5, R7, R12, R23):
  theta_ch   Gamma1 fourth-order part of the CH equation: 1/2 = Crank-Nicolson
             ("Crank-Nicholson and extrapolation for the non-linear terms in R
             and f");
  theta_adv  advection div(phi_n v^n) inside the CH system: 1/2 = Crank-Nicolson;
  theta_visc viscous term of Eq. 19: 1 = implicit at u^{n+1}, the boundary value
             problem "for u^{n+1}" with boundary values of u^{n+1};
  startup_be the first `startup_be` steps (time index n < startup_be) take
             theta_ch = theta_adv = 1 (backward-Euler start-up of the CN scheme
             for the discontinuous initial phi of BASELINE.json, R23).
"""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class Params:
    dt: float = 1e-4
    Gamma1: float = 33.467
    Gamma2: float = 1.25e6
    Lambda: float = 1e-10
    mu: float = 0.14
    Kc: float = 0.15
    eps: float = 1.0
    A: float = 100.0
    Ds: float = 2.3
    Re_s: float = 9.98e-4
    Re_n: float = 2.33e-9
    rho_n: float = 1.0
    rho_s: float = 1.0
    lid_u: float = 1.0
    theta_ch: float = 0.5
    theta_adv: float = 0.5
    theta_visc: float = 1.0
    startup_be: int = 2
    rtol: float = 1e-10
    maxit: int = 200000
    ch_solver: str = "bicgstab"   # "bicgstab" | "gmres"   [R14]
    gmres_restart: int = 30

    def with_(self, **kw) -> "Params":
        return replace(self, **kw)


def nondimensionalise(*, t0: float, h0: float, rho0: float, eta_s: float,
                      eta_n: float, D: float, mu_dim: float, A_dim: float) -> dict:
    """PAPER.md:100-104 (Eq. 15): Re_s = rho0 h^2/(eta_s t0), Re_n = rho0 h^2/(eta_n t0),
    D_s = D t0/h^2, mu~ = mu t0, A~ = A t0.  Pinned against §5's printed values
    computed from Table 1."""
    return dict(
        Re_s=rho0 * h0 ** 2 / (eta_s * t0),
        Re_n=rho0 * h0 ** 2 / (eta_n * t0),
        Ds=D * t0 / h0 ** 2,
        mu=mu_dim * t0,
        A=A_dim * t0,
    )
