"""Assembled sparse operators of the discretisation.  Test infrastructure only.

PAPER.md §4 (lines 142-151): "central differences for the spatial
discretization", uniform grid on Omega = [0,1]^2, periodic in x (§5,
PAPER.md:270), zero-flux / no-slip walls in y (Eq. 23-24, Eq. 19 BC).
PAPER.md §4.1 (lines 207-231): the matrices are entered row by row from
stencils (MatSetValuesStencil, Listing 3), "DMDA maps indices that are too
large or small to the other edge of the domain" for periodic x.  This module
does the same with numpy index arithmetic: one (di, dj, coefficient) entry per
stencil point, periodic wrap in x, and the wall ghost rule folded into the
column index in y (R2-R4):

  * "mirror"  cell-centred scalars (phi, mu, c, p): s[-1-k] = s[k],
              s[ny+k] = s[ny-1-k]  (Eq. 24 on the cell-centred grid, R2);
  * "odd"     u on x-faces (cell-centred in y): homogeneous Dirichlet by odd
              reflection, u[-1] = -u[0], u[ny] = -u[ny-1] (the lid value
              enters the right-hand side separately, R3);
  * "vface"   v on y-faces: v[0] and v[ny] are wall values (= 0), dropped.

Flat index k = j*nx + i (row j = y index, x contiguous).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def _entries(nx, ny, di, dj, coef, kind):
    """COO triplets of one stencil offset applied at every cell (vectorised
    MatSetValuesStencil).  `coef` is a scalar or an (ny, nx) array."""
    J, I = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    C = np.broadcast_to(np.asarray(coef, dtype=np.float64), (ny, nx)).copy()
    ii = (I + di) % nx                      # periodic x
    jj = J + dj
    keep = np.ones_like(C, dtype=bool)
    if kind in ("mirror", "odd"):
        lo, hi = jj < 0, jj >= ny
        jj = np.where(lo, -1 - jj, jj)
        jj = np.where(hi, 2 * ny - 1 - jj, jj)
        if kind == "odd":
            C = np.where(lo | hi, -C, C)
    elif kind == "vface":
        keep = (jj >= 1) & (jj <= ny - 1)
    else:
        raise ValueError(kind)
    rows = (J * nx + I)[keep]
    cols = (jj * nx + ii)[keep]
    return rows, cols, C[keep]


def stencil_matrix(nx, ny, entries, kind):
    """Sum of stencil offsets -> CSR (duplicates from folding are summed)."""
    R, Cc, V = [], [], []
    for di, dj, coef in entries:
        r, c, v = _entries(nx, ny, di, dj, coef, kind)
        R.append(r), Cc.append(c), V.append(v)
    n = nx * ny
    return sp.csr_matrix((np.concatenate(V), (np.concatenate(R), np.concatenate(Cc))),
                         shape=(n, n))


def lap(nx, ny, kind="mirror"):
    """5-point Laplacian Delta_h (Listing 3 pattern, scaled by 1/h^2)."""
    hx2, hy2 = (1.0 / nx) ** 2, (1.0 / ny) ** 2
    ent = [(1, 0, 1 / hx2), (-1, 0, 1 / hx2), (0, 1, 1 / hy2), (0, -1, 1 / hy2),
           (0, 0, -2 / hx2 - 2 / hy2)]
    if kind == "vface":
        # rows j >= 1 only; row 0 is the wall value and gets an all-zero row
        A = stencil_matrix(nx, ny, ent, "vface")
        interior = np.ones(nx * ny)
        interior[:nx] = 0.0
        return (sp.diags(interior) @ A).tocsr()
    return stencil_matrix(nx, ny, ent, kind)


def flux_div(nx, ny, Kx, Ky):
    """L_K s = div_h(K grad_h s) in conservative face form (Eq. 4 /
    Eq. 20 "∇·(λφ∇ δf/δφ)", "-∇·(1/ρ)∇p").
    Kx: (ny, nx), Kx[j, i] on the x-face between cells i-1 and i.
    Ky: (ny+1, nx), Ky[j, i] on the y-face between rows j-1 and j; Ky[0] and
    Ky[ny] are the walls (zero flux, Eq. 23)."""
    hx2, hy2 = (1.0 / nx) ** 2, (1.0 / ny) ** 2
    Kx = np.asarray(Kx, dtype=np.float64)
    Ky = np.asarray(Ky, dtype=np.float64)
    KE = np.roll(Kx, -1, axis=1)       # right face of cell i = Kx[:, i+1]
    KW = Kx
    KN = Ky[1:, :]                     # top face of row j
    KS = Ky[:-1, :]                    # bottom face of row j
    ent = [(1, 0, KE / hx2), (-1, 0, KW / hx2), (0, 1, KN / hy2), (0, -1, KS / hy2),
           (0, 0, -(KE + KW) / hx2 - (KN + KS) / hy2)]
    return stencil_matrix(nx, ny, ent, "mirror")


def mac_div(nx, ny):
    """Discrete divergence D_h from faces to cells (Eq. 1 / Eq. 20 RHS):
    D(u,v)[j,i] = (u[j,i+1]-u[j,i])/hx + (v[j+1,i]-v[j,i])/hy, with the top
    wall face v[ny] = 0 (not stored) and v[0] the stored bottom wall value."""
    n = nx * ny
    hx, hy = 1.0 / nx, 1.0 / ny
    J, I = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    c = (J * nx + I).ravel()
    uE = (J * nx + (I + 1) % nx).ravel()
    uW = c
    rows = [c, c]
    cols = [uE, uW]
    vals = [np.full(n, 1 / hx), np.full(n, -1 / hx)]
    top = (J < ny - 1).ravel()
    rows += [c[top], c]
    cols += [n + (c[top] + nx), n + c]
    vals += [np.full(top.sum(), 1 / hy), np.full(n, -1 / hy)]
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, 2 * n))


def mac_grad(nx, ny):
    """Discrete gradient G_h from cells to faces (Eq. 21 "∇p^{n+1}"):
    x-face (j,i): (p[j,i]-p[j,i-1])/hx;  y-face (j,i), j>=1: (p[j,i]-p[j-1,i])/hy;
    wall y-faces (j = 0): 0 (Neumann, Eq. 20 BC)."""
    n = nx * ny
    hx, hy = 1.0 / nx, 1.0 / ny
    J, I = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    c = (J * nx + I).ravel()
    cW = (J * nx + (I - 1) % nx).ravel()
    inner = (J >= 1).ravel()
    rows = [c, c, n + c[inner], n + c[inner]]
    cols = [c, cW, c[inner], c[inner] - nx]
    vals = [np.full(n, 1 / hx), np.full(n, -1 / hx),
            np.full(inner.sum(), 1 / hy), np.full(inner.sum(), -1 / hy)]
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(2 * n, n))


def advection_matrix(nx, ny, u, v):
    """Conservative central advection s -> div_h(s v) on the MAC grid (Eq. 16
    "∇·(φ_n v)", central differences §4; R12) as a matrix, for
    the implicit (Crank-Nicolson) part of the CH step (R12).  Face values of s
    are arithmetic means; v = 0 on the wall faces (Eq. 22, v·n = 0)."""
    hx, hy = 1.0 / nx, 1.0 / ny
    uW = np.asarray(u, dtype=np.float64)
    uE = np.roll(uW, -1, axis=1)               # u on the right face of cell i
    vS = np.array(v, dtype=np.float64, copy=True)
    vS[0] = 0.0                                 # bottom wall face
    vN = np.zeros_like(vS)
    vN[:-1] = vS[1:]                            # top face of row j (wall at j = ny-1)
    ent = [(1, 0, uE / (2 * hx)), (-1, 0, -uW / (2 * hx)),
           (0, 1, vN / (2 * hy)), (0, -1, -vS / (2 * hy)),
           (0, 0, (uE - uW) / (2 * hx) + (vN - vS) / (2 * hy))]
    return stencil_matrix(nx, ny, ent, "mirror")


def ch_matrix(nx, ny, dt, Gamma1, Mx, My, theta=0.5, theta_adv=0.0, u=None, v=None):
    """Implicit Cahn-Hilliard operator (Eq. 16 4th line with §4's
    Crank-Nicolson, R5, R12):
        A = I/dt + theta Gamma1 L_M Delta_h + theta_adv Adv(.; v^n).
    Nonsymmetric (product of two different symmetric operators, plus the
    skew advection part), 13-point."""
    n = nx * ny
    A = (sp.identity(n, format="csr") / dt
         + (theta * Gamma1) * (flux_div(nx, ny, Mx, My) @ lap(nx, ny, "mirror")))
    if theta_adv != 0.0:
        A = A + theta_adv * advection_matrix(nx, ny, u, v)
    return A.tocsr()


def nutrient_matrix(nx, ny, a_c, Kx, Ky):
    """A_c = diag(a_c) - (1/2) L_K  (nutrient equation, Eq. 16 3rd line, R11). SPD."""
    return (sp.diags(np.ravel(a_c)) - 0.5 * flux_div(nx, ny, Kx, Ky)).tocsr()


def node_flux_div(nx, ny, KW, KE, KS, KN, kind):
    """div_h(K grad_h .) of one velocity component from its four face
    coefficient arrays (explicit.node_fluxes), ghost rule `kind` ("odd": u,
    "vface": v; rows j >= 1 only, row 0 all zero)."""
    hx2, hy2 = (1.0 / nx) ** 2, (1.0 / ny) ** 2
    ent = [(1, 0, KE / hx2), (-1, 0, KW / hx2), (0, 1, KN / hy2), (0, -1, KS / hy2),
           (0, 0, -(KE + KW) / hx2 - (KN + KS) / hy2)]
    A = stencil_matrix(nx, ny, ent, kind)
    if kind == "vface":
        interior = np.ones(nx * ny)
        interior[:nx] = 0.0
        A = sp.diags(interior) @ A
    return A.tocsr()


def u_matrix(nx, ny, a_u, K, theta=1.0):
    """Implicit viscous operator for u (Eq. 19, R6-R7): diag(a_u) - theta div_h(eta grad_h),
    a_u = rho/dt, K = (KW, KE, KS, KN) face coefficients of eta (theta = 1: the
    boundary value problem for u^{n+1} as printed; 1/2: Crank-Nicolson).  SPD."""
    return (sp.diags(np.ravel(a_u)) - theta * node_flux_div(nx, ny, *K, "odd")).tocsr()


def v_matrix(nx, ny, a_v, K, theta=1.0):
    """Same for v on interior y-faces; the wall row j = 0 is an identity row."""
    a = np.array(a_v, dtype=np.float64, copy=True)
    a[0, :] = 1.0
    return (sp.diags(np.ravel(a)) - theta * node_flux_div(nx, ny, *K, "vface")).tocsr()


def poisson_matrix(nx, ny, beta_x, beta_y):
    """Pressure operator -D_h diag(beta) G_h = -L_beta (Eq. 20, beta = 1/rho^{n+1} on faces).
    SPSD with null space = constants (periodic x + Neumann y)."""
    return (-flux_div(nx, ny, beta_x, beta_y)).tocsr()
