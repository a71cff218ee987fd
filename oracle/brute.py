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


def ch_apply(phis, x, dt, Gamma1, Lambda):
    """x/dt + (G1/2) div(Lambda phi* grad(Delta x))  (R5)."""
    w = lap(x)
    return x / dt + 0.5 * Gamma1 * flux_div(face_from_cells(phis, Lambda, clip=True), w)


def poisson_apply(phi1, p, rho_n, rho_s):
    """-div((1/rho) grad p), rho of the face-mean phi (Eq. 20)."""
    def k(kind, j, i):
        if kind == "x":
            m = 0.5 * (S(phi1, j, i - 1) + S(phi1, j, i))
        else:
            m = 0.5 * (S(phi1, j - 1, i) + S(phi1, j, i))
        return 1.0 / (rho_s + m * (rho_n - rho_s))
    return -flux_div(k, p)


def u_apply(a_u, x):
    """a x - 1/2 Delta^0 x for u (odd reflection, homogeneous)."""
    ny, nx = x.shape
    out = np.zeros_like(x)
    for j in range(ny):
        for i in range(nx):
            c = U(x, j, i, 0.0)
            lapx = ((U(x, j, i + 1, 0.0) - 2 * c + U(x, j, i - 1, 0.0)) * nx * nx
                    + (U(x, j + 1, i, 0.0) - 2 * c + U(x, j - 1, i, 0.0)) * ny * ny)
            out[j, i] = a_u[j, i] * c - 0.5 * lapx
    return out


def v_apply(a_v, x):
    """a x - 1/2 Delta^0 x on interior y-faces, identity on the wall row."""
    ny, nx = x.shape
    out = np.zeros_like(x)
    for i in range(nx):
        out[0, i] = x[0, i]
    for j in range(1, ny):
        for i in range(nx):
            c = V(x, j, i)
            lapx = ((V(x, j, i + 1) - 2 * c + V(x, j, i - 1)) * nx * nx
                    + (V(x, j + 1, i) - 2 * c + V(x, j - 1, i)) * ny * ny)
            out[j, i] = a_v[j, i] * c - 0.5 * lapx
    return out


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


def ch_apply_at(phis, x, j, i, dt, Gamma1, Lambda):
    ny, nx = x.shape

    def m(ja, ia, jb, ib):
        return Lambda * max(0.0, 0.5 * (S(phis, ja, ia) + S(phis, jb, ib)))

    wc = lap_at(x, j, i)
    fe = m(j, i, j, i + 1) * (lap_at(x, j, i + 1) - wc)
    fw = m(j, i - 1, j, i) * (wc - lap_at(x, j, i - 1))
    fn = m(j, i, j + 1, i) * (lap_at(x, j + 1, i) - wc) if j + 1 < ny else 0.0
    fs = m(j - 1, i, j, i) * (wc - lap_at(x, j - 1, i)) if j > 0 else 0.0
    return S(x, j, i) / dt + 0.5 * Gamma1 * ((fe - fw) * nx * nx + (fn - fs) * ny * ny)


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
