"""Brute-force scalar-loop stencils for tiny grids.  Test infrastructure only.

An independent second formulation of the same discrete operators, written
cell by cell with an explicit ghost-lookup function per field kind
(R2-R4) instead of the vectorised index folding of assemble.py /
explicit.py.  The pin tests assert the two agree on ragged, non-square grids
(nx != ny), which catches transposed operands, wrong face indexing, wrong
wall folds and hx/hy swaps in either one.  Pure Python: O(n) with a large
constant, use on grids of a few hundred cells.
"""
from __future__ import annotations

import numpy as np


def S(a, j, i):
    """Cell-centred scalar with mirror walls (Eq. 24, R2) and periodic x."""
    ny, nx = a.shape
    i %= nx
    if j < 0:
        j = -1 - j
    elif j >= ny:
        j = 2 * ny - 1 - j
    return float(a[j, i])


def U(a, j, i, lid):
    """u on x-faces: odd reflection (no-slip) at y=0, lid at y=1 (R3)."""
    ny, nx = a.shape
    i %= nx
    if j < 0:
        return -float(a[-1 - j, i])
    if j >= ny:
        return 2.0 * lid - float(a[2 * ny - 1 - j, i])
    return float(a[j, i])


def V(a, j, i):
    """v on y-faces: v = 0 on both wall faces j = 0 and j = ny (R4)."""
    ny, nx = a.shape
    i %= nx
    if j <= 0 or j >= ny:
        return 0.0
    return float(a[j, i])


def lap(s):
    ny, nx = s.shape
    out = np.zeros_like(s)
    for j in range(ny):
        for i in range(nx):
            c = S(s, j, i)
            out[j, i] = ((S(s, j, i + 1) - 2 * c + S(s, j, i - 1)) * nx * nx
                         + (S(s, j + 1, i) - 2 * c + S(s, j - 1, i)) * ny * ny)
    return out


def flux_div(kface, s):
    """div(K grad s) with K on faces given by callables kface(kind, j, i):
    kind 'x' -> face between (j,i-1),(j,i); kind 'y' -> between (j-1,i),(j,i)."""
    ny, nx = s.shape
    out = np.zeros_like(s)
    for j in range(ny):
        for i in range(nx):
            c = S(s, j, i)
            fe = kface("x", j, i + 1) * (S(s, j, i + 1) - c)
            fw = kface("x", j, i) * (c - S(s, j, i - 1))
            fn = kface("y", j + 1, i) * (S(s, j + 1, i) - c) if j + 1 < ny else 0.0
            fs = kface("y", j, i) * (c - S(s, j - 1, i)) if j > 0 else 0.0
            out[j, i] = (fe - fw) * nx * nx + (fn - fs) * ny * ny
    return out


def face_from_cells(w, scale=1.0, clip=False):
    """K on faces as scale * mean of the two adjacent cell values of w."""
    def k(kind, j, i):
        if kind == "x":
            m = 0.5 * (S(w, j, i - 1) + S(w, j, i))
        else:
            m = 0.5 * (S(w, j - 1, i) + S(w, j, i))
        if clip:
            m = max(0.0, m)
        return scale * m
    return k


def ch_apply(phis, x, dt, Gamma1, Lambda, theta=0.5, theta_adv=0.0, u=None, v=None):
    """x/dt + theta G1 div(Lambda phi* grad(Delta x)) + theta_adv div(x v)  (R5, R12)."""
    w = lap(x)
    out = x / dt + theta * Gamma1 * flux_div(face_from_cells(phis, Lambda, clip=True), w)
    if theta_adv != 0.0:
        out = out + theta_adv * advection(x, u, v)
    return out


def poisson_apply(phi1, p, rho_n, rho_s):
    """-div((1/rho) grad p), rho of the face-mean phi (Eq. 20)."""
    def k(kind, j, i):
        if kind == "x":
            m = 0.5 * (S(phi1, j, i - 1) + S(phi1, j, i))
        else:
            m = 0.5 * (S(phi1, j - 1, i) + S(phi1, j, i))
        return 1.0 / (rho_s + m * (rho_n - rho_s))
    return -flux_div(k, p)


def _kmean(w, ja, ia, jb, ib):
    """Mean of a node coefficient at two unknown points (mirror rows, periodic x)."""
    return 0.5 * (S(w, ja, ia) + S(w, jb, ib))


def u_apply(a_u, eta, x, theta=1.0):
    """a x - theta div(eta grad x) for u (odd reflection, homogeneous), face
    coefficient = mean of eta at the two u points."""
    ny, nx = x.shape
    out = np.zeros_like(x)
    for j in range(ny):
        for i in range(nx):
            c = U(x, j, i, 0.0)
            fe = _kmean(eta, j, i, j, i + 1) * (U(x, j, i + 1, 0.0) - c)
            fw = _kmean(eta, j, i - 1, j, i) * (c - U(x, j, i - 1, 0.0))
            fn = _kmean(eta, j, i, j + 1, i) * (U(x, j + 1, i, 0.0) - c)
            fs = _kmean(eta, j - 1, i, j, i) * (c - U(x, j - 1, i, 0.0))
            out[j, i] = a_u[j, i] * c - theta * ((fe - fw) * nx * nx + (fn - fs) * ny * ny)
    return out


def v_apply(a_v, eta, x, theta=1.0):
    """a x - theta div(eta grad x) on interior y-faces, identity on the wall row."""
    ny, nx = x.shape
    out = np.zeros_like(x)
    for i in range(nx):
        out[0, i] = x[0, i]
    for j in range(1, ny):
        for i in range(nx):
            c = V(x, j, i)
            fe = _kmean(eta, j, i, j, i + 1) * (V(x, j, i + 1) - c)
            fw = _kmean(eta, j, i - 1, j, i) * (c - V(x, j, i - 1))
            fn = _kmean(eta, j, i, j + 1, i) * (V(x, j + 1, i) - c)
            fs = _kmean(eta, j - 1, i, j, i) * (c - V(x, j - 1, i))
            out[j, i] = a_v[j, i] * c - theta * ((fe - fw) * nx * nx + (fn - fs) * ny * ny)
    return out


def visc_transpose(u, v, phis, Re_n, Re_s):
    """div(eta (grad v)^T) on the MAC faces, eta(phi) = f/Re_n + (1-f)/Re_s,
    f = clip(phi, 0, 1), at cell centres and at corners (phi = mean of the
    four cells, mirror rows)."""
    ny, nx = u.shape

    def eta(p):
        f = min(max(p, 0.0), 1.0)
        return f / Re_n + (1.0 - f) / Re_s

    eta_cell = np.array([[eta(phis[j, i]) for i in range(nx)] for j in range(ny)])

    def ek(j, i):  # corner (i hx, j hy)
        return eta(0.25 * (S(phis, j, i) + S(phis, j, i - 1) + S(phis, j - 1, i)
                           + S(phis, j - 1, i - 1)))

    tx = np.zeros_like(u)
    ty = np.zeros_like(v)
    for j in range(ny):
        for i in range(nx):
            qe = S(eta_cell, j, i) * (U(u, j, i + 1, 0.0) - U(u, j, i, 0.0)) * nx
            qw = S(eta_cell, j, i - 1) * (U(u, j, i, 0.0) - U(u, j, i - 1, 0.0)) * nx
            rn = ek(j + 1, i) * (V(v, j + 1, i) - V(v, j + 1, i - 1)) * nx
            rs = ek(j, i) * (V(v, j, i) - V(v, j, i - 1)) * nx
            tx[j, i] = (qe - qw) * nx + (rn - rs) * ny
    for j in range(1, ny):
        for i in range(nx):
            qe = ek(j, i + 1) * (U(u, j, i + 1, 0.0) - U(u, j - 1, i + 1, 0.0)) * ny
            qw = ek(j, i) * (U(u, j, i, 0.0) - U(u, j - 1, i, 0.0)) * ny
            rn = S(eta_cell, j, i) * (V(v, j + 1, i) - V(v, j, i)) * ny
            rs = S(eta_cell, j - 1, i) * (V(v, j, i) - V(v, j - 1, i)) * ny
            ty[j, i] = (qe - qw) * nx + (rn - rs) * ny
    return tx, ty


def divergence(u, v):
    ny, nx = u.shape
    out = np.zeros_like(u)
    for j in range(ny):
        for i in range(nx):
            out[j, i] = ((U(u, j, i + 1, 0.0) - U(u, j, i, 0.0)) * nx
                         + (V(v, j + 1, i) - V(v, j, i)) * ny)
    return out


def advection(s, u, v):
    ny, nx = s.shape
    out = np.zeros_like(s)
    for j in range(ny):
        for i in range(nx):
            c = S(s, j, i)
            fe = U(u, j, i + 1, 0.0) * 0.5 * (c + S(s, j, i + 1))
            fw = U(u, j, i, 0.0) * 0.5 * (c + S(s, j, i - 1))
            fn = V(v, j + 1, i) * 0.5 * (c + S(s, j + 1, i))
            fs = V(v, j, i) * 0.5 * (c + S(s, j - 1, i))
            out[j, i] = (fe - fw) * nx + (fn - fs) * ny
    return out


def convective(u, v, lid):
    ny, nx = u.shape
    cu = np.zeros_like(u)
    cv = np.zeros_like(v)
    for j in range(ny):
        for i in range(nx):
            vbar = 0.25 * (V(v, j, i - 1) + V(v, j, i) + V(v, j + 1, i - 1) + V(v, j + 1, i))
            cu[j, i] = (U(u, j, i, lid) * (U(u, j, i + 1, lid) - U(u, j, i - 1, lid)) * nx / 2
                        + vbar * (U(u, j + 1, i, lid) - U(u, j - 1, i, lid)) * ny / 2)
    for j in range(1, ny):
        for i in range(nx):
            ubar = 0.25 * (U(u, j - 1, i, lid) + U(u, j - 1, i + 1, lid)
                           + U(u, j, i, lid) + U(u, j, i + 1, lid))
            cv[j, i] = (ubar * (V(v, j, i + 1) - V(v, j, i - 1)) * nx / 2
                        + V(v, j, i) * (V(v, j + 1, i) - V(v, j - 1, i)) * ny / 2)
    return cu, cv


def phase_stress(phis, Gamma1):
    ny, nx = phis.shape

    def txx(j, i):
        return ((S(phis, j, i + 1) - S(phis, j, i - 1)) * nx / 2) ** 2

    def tyy(j, i):
        return ((S(phis, j + 1, i) - S(phis, j - 1, i)) * ny / 2) ** 2

    def txy(j, i):  # corner at (i hx, j hy)
        a, b = S(phis, j, i), S(phis, j - 1, i)
        c, d = S(phis, j, i - 1), S(phis, j - 1, i - 1)
        return ((a + b - c - d) * nx / 2) * ((a + c - b - d) * ny / 2)

    rx = np.zeros_like(phis)
    ry = np.zeros_like(phis)
    for j in range(ny):
        for i in range(nx):
            rx[j, i] = -Gamma1 * ((txx(j, i) - txx(j, i - 1)) * nx
                                  + (txy(j + 1, i) - txy(j, i)) * ny)
    for j in range(1, ny):
        for i in range(nx):
            ry[j, i] = -Gamma1 * ((txy(j, i + 1) - txy(j, i)) * nx
                                  + (tyy(j, i) - tyy(j - 1, i)) * ny)
    return rx, ry


# ----------------------------------------------------- single-cell versions
# For sampled checks at full size (4096^2): O(1) work per requested cell.
def lap_at(s, j, i):
    ny, nx = s.shape
    c = S(s, j, i)
    return ((S(s, j, i + 1) - 2 * c + S(s, j, i - 1)) * nx * nx
            + (S(s, j + 1, i) - 2 * c + S(s, j - 1, i)) * ny * ny)


def ch_apply_at(phis, x, j, i, dt, Gamma1, Lambda, theta=0.5, theta_adv=0.0, u=None, v=None):
    ny, nx = x.shape

    def m(ja, ia, jb, ib):
        return Lambda * max(0.0, 0.5 * (S(phis, ja, ia) + S(phis, jb, ib)))

    wc = lap_at(x, j, i)
    fe = m(j, i, j, i + 1) * (lap_at(x, j, i + 1) - wc)
    fw = m(j, i - 1, j, i) * (wc - lap_at(x, j, i - 1))
    fn = m(j, i, j + 1, i) * (lap_at(x, j + 1, i) - wc) if j + 1 < ny else 0.0
    fs = m(j - 1, i, j, i) * (wc - lap_at(x, j - 1, i)) if j > 0 else 0.0
    out = S(x, j, i) / dt + theta * Gamma1 * ((fe - fw) * nx * nx + (fn - fs) * ny * ny)
    if theta_adv != 0.0:
        c = S(x, j, i)
        ae = U(u, j, i + 1, 0.0) * 0.5 * (c + S(x, j, i + 1))
        aw = U(u, j, i, 0.0) * 0.5 * (c + S(x, j, i - 1))
        an = V(v, j + 1, i) * 0.5 * (c + S(x, j + 1, i))
        as_ = V(v, j, i) * 0.5 * (c + S(x, j - 1, i))
        out += theta_adv * ((ae - aw) * nx + (an - as_) * ny)
    return out


def poisson_at(phi1, p, j, i, rho_n, rho_s):
    ny, nx = p.shape

    def beta(ja, ia, jb, ib):
        m = 0.5 * (S(phi1, ja, ia) + S(phi1, jb, ib))
        return 1.0 / (rho_s + m * (rho_n - rho_s))

    c = S(p, j, i)
    fe = beta(j, i, j, i + 1) * (S(p, j, i + 1) - c)
    fw = beta(j, i - 1, j, i) * (c - S(p, j, i - 1))
    fn = beta(j, i, j + 1, i) * (S(p, j + 1, i) - c) if j + 1 < ny else 0.0
    fs = beta(j - 1, i, j, i) * (c - S(p, j - 1, i)) if j > 0 else 0.0
    return -((fe - fw) * nx * nx + (fn - fs) * ny * ny)
