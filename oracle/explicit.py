"""Explicit (right-hand-side) terms of the time step, plain numpy.  Test infrastructure only.

Every function works on (ny, nx) fp64 arrays (row j = y).  Ghost values are
built explicitly with the wall rules of DESIGN.md R2-R4 before differencing;
x is periodic ("periodic boundary conditions in the x direction").
"""
from __future__ import annotations

import numpy as np


# ---------------------------------------------------------------- ghost padding
def pad_scalar(s, w):
    """Cell-centred scalar with w ghost layers: mirror about the wall faces in y
    (Eq. 24 on the cell-centred grid, R2), periodic in x."""
    s = np.pad(s, ((w, w), (0, 0)), mode="symmetric")
    return np.pad(s, ((0, 0), (w, w)), mode="wrap")


def pad_u(u, lid_u):
    """u on x-faces with one ghost layer: no-slip bottom u[-1] = -u[0];
    lid top u[ny] = 2*U0 - u[ny-1] (Eq. 19 BC "u|_{y=0}=0, u|_{y=1}=u_0", R3)."""
    g = np.vstack([-u[:1], u, 2.0 * lid_u - u[-1:]])
    return np.pad(g, ((0, 0), (1, 1)), mode="wrap")


def pad_v(v):
    """v on y-faces with one extra row: v[ny] = 0 (top wall face); the row
    below v[0] (never read by the 5-point stencils on rows >= 1) is -v[1]."""
    z = np.zeros_like(v[:1])
    g = np.vstack([-v[1:2], v, z])
    return np.pad(g, ((0, 0), (1, 1)), mode="wrap")


# ------------------------------------------------------------------ CH pieces
def phi_star(phi, phi_prev):
    """Extrapolated state phi* = (3 phi^n - phi^{n-1})/2 (§4 "extrapolation for the
    non-linear terms"; R5)."""
    return 1.5 * phi - 0.5 * phi_prev


def fprime(phi, Gamma2):
    """d/dphi [Gamma2 phi^2 (1-phi)^2] = 2 Gamma2 phi (1-phi)(1-2 phi) (Eq. 16)."""
    return 2.0 * Gamma2 * phi * (1.0 - phi) * (1.0 - 2.0 * phi)


def mobility_faces(phis, Lambda):
    """Face mobility Lambda*phi* (Eq. 4 "λφ_n", R5): arithmetic face average,
    clipped at 0; wall faces carry zero flux (Eq. 23)."""
    ny, nx = phis.shape
    Mx = Lambda * np.maximum(0.0, 0.5 * (np.roll(phis, 1, axis=1) + phis))
    My = np.zeros((ny + 1, nx))
    My[1:ny] = Lambda * np.maximum(0.0, 0.5 * (phis[:-1] + phis[1:]))
    return Mx, My


def advection(s, u, v):
    """Conservative central advection div_h(s v) on the MAC grid (Eq. 16
    "∇·(φ_n v)", central differences §4; R12).  Face values of s are
    arithmetic means; the wall faces carry v = 0."""
    ny, nx = s.shape
    hx, hy = 1.0 / nx, 1.0 / ny
    uE = np.roll(u, -1, axis=1)
    sE = 0.5 * (s + np.roll(s, -1, axis=1))
    sW = 0.5 * (s + np.roll(s, 1, axis=1))
    vN = np.zeros_like(v)
    vN[:-1] = v[1:]
    vS = v.copy()
    vS[0] = 0.0
    sp = pad_scalar(s, 1)
    sN = 0.5 * (s + sp[2:, 1:-1])
    sS = 0.5 * (s + sp[:-2, 1:-1])
    return (uE * sE - u * sW) / hx + (vN * sN - vS * sS) / hy


def volume_fraction(phi):
    """The physical volume fraction clip(phi, 0, 1) at which the material laws
    and rates of phi_n are evaluated ("volume fraction",
    PAPER.md:42 phi_n + phi_s = 1; R24).  The discrete phi leaves [0, 1] by
    the dispersive ripples of the central scheme."""
    return np.clip(phi, 0.0, 1.0)


def growth(phis, c, eps, mu, Kc):
    """g_n = eps mu phi_n c/(K_c + c) (Eq. 5; "c'" read as c, R8),
    phi_n the volume fraction (R24)."""
    return eps * mu * volume_fraction(phis) * c / (Kc + c)


# ------------------------------------------------------------ momentum pieces
def face_phi_u(phis):
    """phi interpolated to x-faces: (phi[j,i-1] + phi[j,i])/2."""
    return 0.5 * (np.roll(phis, 1, axis=1) + phis)


def face_phi_v(phis):
    """phi interpolated to y-faces j >= 1: (phi[j-1,i] + phi[j,i])/2; row 0
    (the wall) gets phi[0] (never used: v[0] is pinned)."""
    out = phis.copy()
    out[1:] = 0.5 * (phis[:-1] + phis[1:])
    return out


def density(phi, rho_n, rho_s):
    """rho~ = phi_s rho_s/rho0 + phi_n rho_n/rho0 (Eq. 15), at the
    volume fraction clip(phi, 0, 1) (R24)."""
    f = volume_fraction(phi)
    return rho_s + f * (rho_n - rho_s)


def inv_reynolds(phi, Re_n, Re_s):
    """1/Re_a = phi_n/Re_n + phi_s/Re_s, the volume-fraction average that makes
    phi_n tau_n + phi_s tau_s = (2/Re_a) D (Eq. 8, Eq. 17; R6), at the volume
    fraction clip(phi, 0, 1) (R24: with Re_n/Re_s = 2.3e-6 any phi below
    -2.3e-6 would make the mixture viscosity negative)."""
    f = volume_fraction(phi)
    return f / Re_n + (1.0 - f) / Re_s


def convective_u(u, v, lid_u):
    """(v·∇u) at x-faces (Eq. 19 "-v^n·∇v^n", central, R7)."""
    ny, nx = u.shape
    hx, hy = 1.0 / nx, 1.0 / ny
    up = pad_u(u, lid_u)
    dudx = (up[1:-1, 2:] - up[1:-1, :-2]) / (2 * hx)
    dudy = (up[2:, 1:-1] - up[:-2, 1:-1]) / (2 * hy)
    vp = pad_v(v)                     # rows: -1, 0..ny-1, ny
    vb = vp[1:-1, :]                  # v[j, i-1..i+1] for rows 0..ny-1
    vt = vp[2:, :]                    # v[j+1, ...]
    vbar = 0.25 * (vb[:, :-2] + vb[:, 1:-1] + vt[:, :-2] + vt[:, 1:-1])
    return u * dudx + vbar * dudy


def convective_v(u, v):
    """(v·∇v) at interior y-faces (row 0 = wall -> 0)."""
    ny, nx = u.shape
    hx, hy = 1.0 / nx, 1.0 / ny
    vp = pad_v(v)
    dvdx = (vp[1:-1, 2:] - vp[1:-1, :-2]) / (2 * hx)
    dvdy = (vp[2:, 1:-1] - vp[:-2, 1:-1]) / (2 * hy)
    uE = np.roll(u, -1, axis=1)
    ubar = np.zeros_like(u)
    ubar[1:] = 0.25 * (u[:-1] + uE[:-1] + u[1:] + uE[1:])
    out = ubar * dvdx + v * dvdy
    out[0] = 0.0
    return out


def phase_stress(phis, Gamma1):
    """R = -Gamma1 ∇·(∇φ ⊗ ∇φ) (Eq. 17; its viscous part vanishes identically
    under R6) on the MAC faces, conservative: cell-centred T_xx, T_yy and
    corner T_xy, each from central differences of phi* with mirror ghosts.
    Returns (R_x on x-faces, R_y on y-faces with row 0 = 0)."""
    ny, nx = phis.shape
    hx, hy = 1.0 / nx, 1.0 / ny
    p = pad_scalar(phis, 1)           # (ny+2, nx+2), p[j+1, i+1] = phi[j, i]
    Txx = ((p[1:-1, 2:] - p[1:-1, :-2]) / (2 * hx)) ** 2
    Tyy = ((p[2:, 1:-1] - p[:-2, 1:-1]) / (2 * hy)) ** 2
    # corners (x = i hx, y = j hy), j = 0..ny, i = 0..nx-1
    a = p[1:, 1:-1]     # phi[j, i]      (rows j = 0..ny  -> padded rows 1..ny+1)
    b = p[:-1, 1:-1]    # phi[j-1, i]
    cW = p[1:, :-2]     # phi[j, i-1]
    dW = p[:-1, :-2]    # phi[j-1, i-1]
    gx = (a + b - cW - dW) / (2 * hx)
    gy = (a + cW - b - dW) / (2 * hy)
    Txy = gx * gy                      # (ny+1, nx)
    Rx = -Gamma1 * ((Txx - np.roll(Txx, 1, axis=1)) / hx + (Txy[1:] - Txy[:-1]) / hy)
    Ry = np.zeros_like(phis)
    Ry[1:] = -Gamma1 * ((np.roll(Txy, -1, axis=1)[1:ny] - Txy[1:ny]) / hx
                        + (Tyy[1:] - Tyy[:-1]) / hy)
    return Rx, Ry


def viscosity_u(phis, Re_n, Re_s):
    """eta = 1/Re_a (R6, R24) at the u points (x-faces), from the face mean of phi*."""
    return inv_reynolds(face_phi_u(phis), Re_n, Re_s)


def viscosity_v(phis, Re_n, Re_s):
    """eta at the v points (y-faces j >= 1; row 0, the wall, from phi[0])."""
    return inv_reynolds(face_phi_v(phis), Re_n, Re_s)


def node_fluxes(w):
    """Face coefficients of div(w grad .) between adjacent unknown points of one
    velocity component, K = arithmetic mean of w at the two points (R6): returns
    (KW, KE, KS, KN), KW[j, i] between points (j, i-1) and (j, i), KS[j, i]
    between (j-1, i) and (j, i); the coefficient's wall ghost is its mirror
    image (KS[0] = w[0], KN[ny-1] = w[ny-1])."""
    KW = 0.5 * (np.roll(w, 1, axis=1) + w)
    KE = np.roll(KW, -1, axis=1)
    wp = np.vstack([w[:1], w, w[-1:]])
    KS = 0.5 * (wp[:-2] + wp[1:-1])
    KN = 0.5 * (wp[2:] + wp[1:-1])
    return KW, KE, KS, KN


def visc_u_inhom(u, eta_u, lid_u):
    """div_h(eta grad_h u) at the u points with the no-slip / lid ghosts
    (inhomogeneous; the viscous term of Eq. 18-19 in conservative form, R6)."""
    ny, nx = u.shape
    up = pad_u(u, lid_u)
    KW, KE, KS, KN = node_fluxes(eta_u)
    return ((KE * (up[1:-1, 2:] - u) - KW * (u - up[1:-1, :-2])) * nx * nx
            + (KN * (up[2:, 1:-1] - u) - KS * (u - up[:-2, 1:-1])) * ny * ny)


def visc_v(v, eta_v):
    """div_h(eta grad_h v) on interior y-faces with v = 0 on both walls; row 0 -> 0."""
    ny, nx = v.shape
    vp = pad_v(v)
    KW, KE, KS, KN = node_fluxes(eta_v)
    out = ((KE * (vp[1:-1, 2:] - v) - KW * (v - vp[1:-1, :-2])) * nx * nx
           + (KN * (vp[2:, 1:-1] - v) - KS * (v - vp[:-2, 1:-1])) * ny * ny)
    out[0] = 0.0
    return out


def visc_transpose(u, v, phis, Re_n, Re_s):
    """The rest of the viscous stress, div(eta (grad v)^T), so that with the
    implicit div(eta grad v) the momentum equation carries div(2 eta D) =
    div(phi_n tau_n + phi_s tau_s) (Eq. 8-9, 15; R6: Eq. 17's viscous part of
    R).  MAC discretisation: eta at cell centres (d u/dx, d v/dy there) and at
    corners (mean of the four cells, mirror rows; d v/dx, d u/dy there).
    Returns (T_x on x-faces, T_y on y-faces with row 0 = 0)."""
    ny, nx = u.shape
    hx, hy = 1.0 / nx, 1.0 / ny
    ec = inv_reynolds(phis, Re_n, Re_s)
    p = np.pad(phis, ((1, 1), (0, 0)), mode="symmetric")
    pk = 0.25 * (p[1:] + np.roll(p[1:], 1, axis=1) + p[:-1] + np.roll(p[:-1], 1, axis=1))
    ek = inv_reynolds(pk, Re_n, Re_s)                   # corners (i hx, j hy), j = 0..ny
    vf = np.vstack([v, np.zeros((1, nx))])               # v[ny] = 0 (top wall)
    vf[0] = 0.0                                          # bottom wall
    qc = ec * (np.roll(u, -1, axis=1) - u) / hx          # eta du/dx at cells
    dvdx = (vf - np.roll(vf, 1, axis=1)) / hx            # dv/dx at corners
    Tx = (qc - np.roll(qc, 1, axis=1)) / hx + (ek[1:] * dvdx[1:] - ek[:-1] * dvdx[:-1]) / hy
    dudy = np.zeros((ny + 1, nx))
    dudy[1:ny] = (u[1:] - u[:-1]) / hy                   # du/dy at interior corners
    qk = ek * dudy
    rc = ec * (vf[1:] - vf[:-1]) / hy                    # eta dv/dy at cells
    Ty = np.zeros_like(v)
    Ty[1:] = (np.roll(qk, -1, axis=1) - qk)[1:ny] / hx + (rc[1:] - rc[:-1]) / hy
    return Tx, Ty


# ----------------------------------------------------------- projection pieces
def divergence(u, v):
    """D_h(u, v) at cells (Eq. 1 / Eq. 20 RHS), v[ny] = 0, v[0] = wall value."""
    ny, nx = u.shape
    vN = np.zeros_like(v)
    vN[:-1] = v[1:]
    vS = v.copy()
    vS[0] = 0.0
    return (np.roll(u, -1, axis=1) - u) * nx + (vN - vS) * ny


def pressure_faces(phi1, rho_n, rho_s):
    """beta = 1/rho^{n+1} on faces (Eq. 20 "1/ρ^{n+1}"), rho of the face-averaged
    phi (rho is affine in phi).  Wall y-faces: 0 (Neumann, Eq. 20 BC)."""
    ny, nx = phi1.shape
    bx = 1.0 / density(face_phi_u(phi1), rho_n, rho_s)
    by = np.zeros((ny + 1, nx))
    by[1:ny] = 1.0 / density(0.5 * (phi1[:-1] + phi1[1:]), rho_n, rho_s)
    return bx, by


def correct(us, vs, p, bx, by):
    """v^{n+1} = u^{n+1} + (1/ρ^{n+1}) ∇p^{n+1} (Eq. 21), MAC faces."""
    ny, nx = p.shape
    u1 = us + bx * (p - np.roll(p, 1, axis=1)) * nx
    v1 = vs.copy()
    v1[1:] = vs[1:] + by[1:ny] * (p[1:] - p[:-1]) * ny
    v1[0] = 0.0
    return u1, v1


# ---------------------------------------------------------------- diagnostics
def mass(phi):
    """∫ phi_n dx over the unit square (midpoint rule)."""
    return float(phi.sum()) / phi.size


def free_energy(phi, Gamma1, Gamma2):
    """Discrete f of Eq. 16 integrated over Omega:
    hx hy [Gamma1/2 (sum of squared face differences / h^2, interior faces
    + periodic x) + Gamma2 sum phi^2 (1-phi)^2].  The gradient part equals
    -Gamma1/2 <phi, Delta_h phi> for the mirror Laplacian (summation by parts)."""
    ny, nx = phi.shape
    dx = (phi - np.roll(phi, 1, axis=1)) * nx
    dy = (phi[1:] - phi[:-1]) * ny
    grad2 = (dx ** 2).sum() + (dy ** 2).sum()
    bulk = (phi ** 2 * (1 - phi) ** 2).sum()
    return float((0.5 * Gamma1 * grad2 + Gamma2 * bulk) / (nx * ny))
