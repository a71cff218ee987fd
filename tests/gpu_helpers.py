"""Shared helpers of the GPU parity tests (test infrastructure: they call the
C ABI through the binding and the CPU oracle side by side)."""
import numpy as np

FIELDS = ("phi", "c", "u", "v", "p")


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0))


def oracle_params(sp, **kw):
    """oracle.Params with the same values as the binding's SimParams."""
    from oracle import Params
    d = dict(dt=sp.dt, Gamma1=sp.Gamma1, Gamma2=sp.Gamma2, Lambda=sp.Lambda, mu=sp.mu, Kc=sp.Kc,
             eps=sp.eps, A=sp.A, Ds=sp.Ds, Re_s=sp.Re_s, Re_n=sp.Re_n, rho_n=sp.rho_n,
             rho_s=sp.rho_s, lid_u=sp.lid_u, rtol=sp.rtol, maxit=sp.maxit,
             ch_solver=sp.ch_solver, gmres_restart=sp.gmres_restart, theta_ch=sp.theta_ch,
             theta_adv=sp.theta_adv, theta_visc=sp.theta_visc, startup_be=sp.startup_be)
    d.update(kw)
    return Params(**d)


def stream_velocity(nx, ny, seed, scale):
    """Discretely divergence-free MAC velocity (u on x-faces, v on y-faces,
    v = 0 on the walls) from a smooth random corner stream function that
    vanishes on both walls; |u| ~ scale."""
    rng = np.random.default_rng(seed)
    x = np.arange(nx) / nx
    y = np.arange(ny + 1) / ny
    X, Y = np.meshgrid(x, y)
    psi = np.zeros_like(X)
    for _ in range(4):
        k, l = rng.integers(1, 4), rng.integers(1, 4)
        a, ph = rng.standard_normal(), rng.random() * 2 * np.pi
        psi += a * np.sin(l * np.pi * Y) * np.cos(2 * np.pi * k * X + ph) / (k + l)
    psi *= scale / 10.0
    u = (psi[1:] - psi[:-1]) * ny
    v = -(np.roll(psi, -1, axis=1) - psi)[:ny] * nx
    v[0] = 0.0
    return np.ascontiguousarray(u), np.ascontiguousarray(v)


def run_both(nx, ny, steps, seed=0, slabs=1, fields=None, **over):
    """Run `steps` GPU steps and `steps` oracle steps from the same inputs."""
    from paper_1811_11842_b200 import SimParams, Simulation
    from oracle import initial_state, step
    from workloads import initial_fields
    f = fields if fields is not None else initial_fields(nx, ny, seed=seed)
    sp = SimParams(**over)
    sim = Simulation(nx, ny, sp, virtual_slabs=slabs)
    sim.set_fields(**f)
    sim.step(steps)
    got = sim.get_fields(FIELDS + ("u_star", "v_star"))
    st = sim.stats()
    sim.close()
    ost = initial_state(f)
    prm = oracle_params(sp)
    iters = []
    for _ in range(steps):
        ost, info = step(ost, prm)
        iters.append(info.iters)
    gu, gv = ost.guess_uv()   # u*, v* of the last step (R25)
    ref = dict(phi=ost.phi, c=ost.c, u=ost.u, v=ost.v, p=ost.p, u_star=gu, v_star=gv)
    return got, ref, st, iters
