"""Textbook Krylov solvers with a Jacobi preconditioner.  Test infrastructure only.

PAPER.md §4.1 (lines 233-252): "GMRES with a Jacobi preconditioner",
"KSPSolve(ksp,b,x)", and for the singular all-Neumann/periodic pressure
system "we use PETSc to remove the null space of constant functions"
(Listing 5).  BASELINE.json north_star adds BiCGStab for the nonsymmetric CH
system and CG for the symmetric ones.  Stopping rule for all three (R13):
||b - A x_k||_2 <= rtol * ||b||_2 on the method's own residual (CG/BiCGStab:
recursively updated residual; GMRES: the Givens least-squares residual);
b = 0 returns x = 0.  Library primitives used: sparse matvec, dot, norm,
triangular solve -- nothing else.
"""
from __future__ import annotations

import numpy as np


class NotConverged(RuntimeError):
    pass


def _norm(x):
    return float(np.sqrt(np.dot(x, x)))


def cg(A, b, x0, dinv, rtol, maxit, nullspace=False):
    """Preconditioned conjugate gradients (Hestenes-Stiefel), z = D^{-1} r.
    nullspace=True: b is projected onto mean-zero (MatNullSpaceRemove, Listing 5)
    and the returned x has zero mean."""
    b = np.array(b, dtype=np.float64, copy=True)
    if nullspace:
        b -= b.mean()
    bn = _norm(b)
    if bn == 0.0:
        return np.zeros_like(b), 0
    tol = rtol * bn
    x = np.array(x0, dtype=np.float64, copy=True)
    r = b - A @ x
    it = 0
    if _norm(r) > tol:
        z = dinv * r
        p = z.copy()
        rz = float(np.dot(r, z))
        while True:
            it += 1
            q = A @ p
            alpha = rz / float(np.dot(p, q))
            x += alpha * p
            r -= alpha * q
            if _norm(r) <= tol:
                break
            if it >= maxit:
                raise NotConverged(f"cg: {it} iterations, |r|/|b| = {_norm(r) / bn:.3e}")
            z = dinv * r
            rz_new = float(np.dot(r, z))
            beta = rz_new / rz
            rz = rz_new
            p = z + beta * p
    if nullspace:
        x -= x.mean()
    return x, it


def bicgstab(A, b, x0, dinv, rtol, maxit):
    """Right-preconditioned BiCGStab (van der Vorst 1992), p^ = D^{-1} p."""
    b = np.asarray(b, dtype=np.float64)
    bn = _norm(b)
    if bn == 0.0:
        return np.zeros_like(b), 0
    tol = rtol * bn
    x = np.array(x0, dtype=np.float64, copy=True)
    r = b - A @ x
    it = 0
    if _norm(r) <= tol:
        return x, 0
    rhat = r.copy()
    rho_old = alpha = omega = 1.0
    v = np.zeros_like(b)
    p = np.zeros_like(b)
    while True:
        it += 1
        rho = float(np.dot(rhat, r))
        if rho == 0.0:
            raise NotConverged("bicgstab: breakdown rho = 0")
        beta = (rho / rho_old) * (alpha / omega)
        p = r + beta * (p - omega * v)
        phat = dinv * p
        v = A @ phat
        alpha = rho / float(np.dot(rhat, v))
        s = r - alpha * v
        if _norm(s) <= tol:
            x += alpha * phat
            break
        shat = dinv * s
        t = A @ shat
        omega = float(np.dot(t, s)) / float(np.dot(t, t))
        x += alpha * phat + omega * shat
        r = s - omega * t
        if _norm(r) <= tol:
            break
        if it >= maxit:
            raise NotConverged(f"bicgstab: {it} iterations, |r|/|b| = {_norm(r) / bn:.3e}")
        rho_old = rho
    return x, it


def gmres(A, b, x0, dinv, rtol, maxit, restart=30):
    """Restarted right-preconditioned GMRES(m): Arnoldi with modified
    Gram-Schmidt, Givens rotations on the Hessenberg matrix (Saad & Schultz)."""
    b = np.asarray(b, dtype=np.float64)
    bn = _norm(b)
    if bn == 0.0:
        return np.zeros_like(b), 0
    tol = rtol * bn
    x = np.array(x0, dtype=np.float64, copy=True)
    n = b.size
    m = restart
    total = 0
    while True:
        r = b - A @ x
        beta = _norm(r)
        if beta <= tol:
            return x, total
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            total += 1
            w = A @ (dinv * V[j])
            for i in range(j + 1):                       # modified Gram-Schmidt
                H[i, j] = float(np.dot(w, V[i]))
                w -= H[i, j] * V[i]
            H[j + 1, j] = _norm(w)
            if H[j + 1, j] != 0.0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                           # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            if abs(g[j + 1]) <= tol or total >= maxit:
                break
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):                   # back substitution
            y[i] = (g[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]
        x += dinv * (V[:k].T @ y)
        if abs(g[k]) <= tol:
            return x, total
        if total >= maxit:
            raise NotConverged(f"gmres: {total} iterations, est |r|/|b| = {abs(g[k]) / bn:.3e}")
