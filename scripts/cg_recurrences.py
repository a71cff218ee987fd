"""Attainable accuracy of three CG recurrences (R22), numpy, CPU.

Jacobi-preconditioned CG on a 1-D variable-coefficient SPD tridiagonal
system, stopped on the recursive residual at rtol; prints the TRUE relative
residual at the stop for
  hs     Hestenes-Stiefel (the oracle's algorithm),
  cg3    three-term recurrence for both z and x (Concus-Golub-O'Leary),
  cg3x2  three-term z recurrence, two-term p/x updates (the GPU default).
    python scripts/cg_recurrences.py [--n 16000]
"""
import argparse

import numpy as np
import scipy.sparse as sp


def hs(A, b, x0, d, rtol, maxit):
    x = x0.copy()
    r = b - A @ x
    z = r / d
    p = z.copy()
    g = r @ z
    bn = np.linalg.norm(b)
    for k in range(maxit):
        if np.linalg.norm(r) <= rtol * bn:
            return x, k
        q = A @ p
        a = g / (p @ q)
        x += a * p
        r -= a * q
        z = r / d
        gn = r @ z
        p = z + (gn / g) * p
        g = gn
    return x, maxit


def cg3(A, b, x0, d, rtol, maxit, two_term_x):
    bn = np.linalg.norm(b)
    x = x0.copy()
    z = (b - A @ x) / d
    xp, zp = x.copy(), z.copy()
    mu, nu = z @ (d * z), z @ (A @ z)
    om = 1.0
    gp = mup = al = None
    p = np.zeros_like(x)
    for k in range(maxit):
        if np.linalg.norm(d * z) <= rtol * bn:
            return x, k
        gam = mu / nu
        om = 1.0 if k == 0 else 1.0 / (1.0 - (gam / gp) * (mu / mup) / om)
        if two_term_x:  # Chronopoulos-Gear alpha, beta from the same mu, nu
            be = 0.0 if k == 0 else mu / mup
            al = mu / nu if k == 0 else mu / (nu - be * mu / al)
            p = z + be * p
            x = x + al * p
        else:
            x, xp = om * (x + gam * z) + (1 - om) * xp, x
        zn = om * (z - gam * (A @ z) / d) + (1 - om) * zp
        zp, z = z, zn
        gp, mup = gam, mu
        mu, nu = z @ (d * z), z @ (A @ z)
    return x, maxit


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16000)
    ap.add_argument("--rtol", type=float, default=1e-10)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    k = rng.uniform(0.5, 2.0, a.n + 1)
    A = sp.diags([-k[1:-1], k[:-1] + k[1:], -k[1:-1]], [-1, 0, 1]).tocsr()
    b = rng.standard_normal(a.n)
    x0 = rng.standard_normal(a.n)
    d = A.diagonal()
    bn = np.linalg.norm(b)
    xh, kh = hs(A, b, x0, d, a.rtol, 10 * a.n)
    for name, (x, it) in (("hs", (xh, kh)),
                          ("cg3", cg3(A, b, x0, d, a.rtol, 10 * a.n, False)),
                          ("cg3x2", cg3(A, b, x0, d, a.rtol, 10 * a.n, True))):
        print(f"{name:6s} iters {it:6d}  true rel residual {np.linalg.norm(b - A @ x) / bn:.2e}"
              f"  |x - x_hs|/|x_hs| {np.linalg.norm(x - xh) / np.linalg.norm(xh):.1e}")


if __name__ == "__main__":
    main()
