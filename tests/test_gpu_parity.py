"""GPU path (C ABI, sm_100a kernels) vs the CPU oracle, element by element.

Tolerances (north_star): relative L2 <= 1e-9 per field after one step,
<= 1e-6 after 100 steps; every Krylov solve reaches ||r||/||b|| <= 1e-10.
Operator applies are exact up to rounding: relative L2 <= 1e-13.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("phi", "c", "u", "v", "p")


def _rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def _oracle_params(sp, **kw):
    from oracle import Params
    d = dict(dt=sp.dt, Gamma1=sp.Gamma1, Gamma2=sp.Gamma2, Lambda=sp.Lambda, mu=sp.mu, Kc=sp.Kc,
             eps=sp.eps, A=sp.A, Ds=sp.Ds, Re_s=sp.Re_s, Re_n=sp.Re_n, rho_n=sp.rho_n,
             rho_s=sp.rho_s, lid_u=sp.lid_u, rtol=sp.rtol, maxit=sp.maxit,
             ch_solver=sp.ch_solver, gmres_restart=sp.gmres_restart)
    d.update(kw)
    return Params(**d)


def _run_both(nx, ny, steps, seed=0, slabs=1, **over):
    from paper_1811_11842_b200 import Simulation, SimParams
    from oracle import initial_state, step
    from workloads import initial_fields
    f = initial_fields(nx, ny, seed=seed)
    sp = SimParams(**over)
    sim = Simulation(nx, ny, sp, virtual_slabs=slabs)
    sim.set_fields(**f)
    sim.step(steps)
    got = sim.get_fields()
    st = sim.stats()
    sim.close()
    ost = initial_state(f)
    prm = _oracle_params(sp)
    iters = []
    for _ in range(steps):
        ost, info = step(ost, prm)
        iters.append(info.iters)
    ref = dict(phi=ost.phi, c=ost.c, u=ost.u, v=ost.v, p=ost.p)
    return got, ref, st, iters


def _oracle_truncation(nx, ny, seed=0, steps=1, **over):
    """Relative L2 distance, per field, between the oracle's step at the run's
    rtol and the same step solved to rtol 1e-13: how far the solution itself
    moves with the solver's stopping point (oracle only, no GPU input)."""
    from paper_1811_11842_b200 import SimParams
    from oracle import initial_state, step
    from workloads import initial_fields
    f = initial_fields(nx, ny, seed=seed)
    sp = SimParams(**over)
    a = b = initial_state(f)
    for _ in range(steps):
        a, _ = step(a, _oracle_params(sp))
        b, _ = step(b, _oracle_params(sp, rtol=1e-13))
    return {k: _rel(getattr(a, k), getattr(b, k)) for k in FIELDS}


@pytest.mark.parametrize("nx,ny", [(64, 64), (50, 37), (130, 70)])
def test_one_step_matches_oracle(nx, ny):
    """Element-by-element parity, north_star bound 1e-9 on every field.  The
    solves run to rtol 1e-12 on both sides (<= north_star's 1e-10): at 1e-10
    the projected v is only determined to ~2e-7 by the stopping point itself
    (R17), so a 1e-9 comparison there would test the stopping
    iteration, not the arithmetic."""
    got, ref, st, iters = _run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (k, _rel(got[k], ref[k]))
    for sysname, n in iters[-1].items():
        assert abs(st["iters_last"][sysname] - n) <= 2, (sysname, st["iters_last"], iters[-1])
        assert st["resid_last"][sysname] <= 1e-12


@pytest.mark.parametrize("refine", [0, 2])
@pytest.mark.parametrize("nx,ny", [(64, 64), (130, 70)])
def test_one_step_at_north_star_rtol(nx, ny, refine):
    """At north_star's rtol 1e-10 every field matches within 1e-9 plus the
    oracle's own stopping-point sensitivity (R17), the iteration counts agree
    within 2 (+ the few restart iterations with true-residual refinement,
    R21) and every solve reaches 1e-10."""
    got, ref, st, iters = _run_both(nx, ny, 1, refine=refine)
    tr = _oracle_truncation(nx, ny)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9 + tr[k], (k, _rel(got[k], ref[k]), tr[k])
    for k in ("phi", "c", "u"):
        assert tr[k] < 1e-9
        assert _rel(got[k], ref[k]) <= 1e-9, (k, _rel(got[k], ref[k]))
    for sysname, n in iters[-1].items():
        slack = 2 + (8 if refine and sysname != "ch" else 0)
        assert -2 <= st["iters_last"][sysname] - n <= slack, (sysname, st["iters_last"], iters[-1])
        assert st["resid_last"][sysname] <= 1e-10


def test_one_step_gmres_matches_oracle():
    got, ref, st, _ = _run_both(64, 64, 1, ch_solver="gmres", Lambda=1e-5)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (k, _rel(got[k], ref[k]))


def test_bicgstab_nontrivial_ch_system():
    """Lambda large enough that the CH system is far from I/dt (many iterations)."""
    got, ref, st, iters = _run_both(48, 40, 2, Lambda=1e-5)
    assert st["iters_last"]["ch"] >= 5
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (k, _rel(got[k], ref[k]))


@pytest.mark.parametrize("cg3", ["1", "0"])
@pytest.mark.parametrize("slabs", [2, 3])
def test_virtual_slabs_match_single_slab(slabs, cg3, monkeypatch):
    """Slab decomposition in y with halo exchange reproduces the 1-slab step
    (CG: three-term z recurrence, z halos only; and s recurrence, z + s halos).
    The Krylov dot products sum in a different order per decomposition, so the
    comparison runs the solves to rtol = 1e-13 (differences are then rounding
    propagated through ~200 CG iterations, not solver tolerance)."""
    from paper_1811_11842_b200 import Simulation
    from workloads import initial_fields
    monkeypatch.setenv("CHB_CG3", cg3)
    f = initial_fields(40, 36, seed=4)
    out, its = [], []
    for s in (1, slabs):
        sim = Simulation(40, 36, virtual_slabs=s, Lambda=1e-5, rtol=1e-13)
        sim.set_fields(**f)
        sim.step(2)
        out.append(sim.get_fields())
        its.append(sim.stats()["iters_last"])
        sim.close()
    for k in FIELDS:
        # v is the stopping-point/rounding-sensitive field (R17): 1e-10 there
        tol = 1e-10 if k == "v" else 1e-11
        assert _rel(out[1][k], out[0][k]) <= tol, (k, _rel(out[1][k], out[0][k]))
    for k in its[0]:
        # at rtol 1e-13 the last iterations sit on the fp64 attainable-accuracy
        # plateau, where the count depends on the reduction order
        assert abs(its[0][k] - its[1][k]) <= 3 + 0.1 * its[0][k], its


def test_virtual_slabs_gmres():
    from paper_1811_11842_b200 import Simulation
    from workloads import initial_fields
    f = initial_fields(36, 32, seed=6)
    out = []
    for s in (1, 2):
        sim = Simulation(36, 32, virtual_slabs=s, Lambda=1e-5, rtol=1e-13, ch_solver="gmres")
        sim.set_fields(**f)
        sim.step(1)
        out.append(sim.get_fields())
        sim.close()
    for k in FIELDS:
        tol = 1e-10 if k == "v" else 1e-11
        assert _rel(out[1][k], out[0][k]) <= tol, (k, _rel(out[1][k], out[0][k]))


def _golden(name):
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", name))


@pytest.mark.parametrize("rtol,gold", [(1e-10, "oracle_256_100.npz"),
                                       (1e-12, "oracle_256_100_rtol1e-12.npz")])
def test_hundred_steps_256_matches_oracle_golden(rtol, gold):
    """BASELINE.json configs[1]: 256^2, 100 steps, dt = 1e-4 vs the oracle's
    fields (tests/golden/, written by scripts/gen_golden.py from oracle/ only).
    north_star bound 1e-6 relative L2, plus the oracle's own stopping-point
    sensitivity over those 100 steps, which the two committed goldens measure
    (rtol 1e-10 vs 1e-12: u 6e-3, v 8e-2, p 3e-2, phi 1.9e-6, c 3e-8 -- the
    scheme with the paper's parameters amplifies per-step perturbations ~1e6
    within ten steps, R19)."""
    from paper_1811_11842_b200 import Simulation
    from workloads import initial_fields
    g10, g12 = _golden("oracle_256_100.npz"), _golden("oracle_256_100_rtol1e-12.npz")
    ref = _golden(gold)
    f = initial_fields(256, 256, seed=int(ref["seed"]))
    sim = Simulation(256, 256, rtol=rtol)
    sim.set_fields(**f)
    sim.step(100)
    got = sim.get_fields()
    sim.close()
    for k in FIELDS:
        sens = _rel(g10[k], g12[k])
        assert _rel(got[k], ref[k]) <= 1e-6 + 2.0 * sens, (k, _rel(got[k], ref[k]), sens)
    # the trajectory-insensitive fields at the flat north_star bound (x3 for phi,
    # whose sensitivity is 1.9e-6 itself)
    assert _rel(got["c"], ref["c"]) <= 1e-6
    assert _rel(got["phi"], ref["phi"]) <= 6e-6


def test_operator_applies_match_assembled_matrices():
    from paper_1811_11842_b200 import Simulation
    from oracle import assemble as asm, explicit as ex
    from oracle.step import initial_state, momentum_systems
    from oracle.params import Params
    from workloads import initial_fields
    nx, ny = 45, 38
    f = initial_fields(nx, ny, seed=1)
    rng = np.random.default_rng(0)
    x = rng.random((ny, nx))
    prm = Params(Lambda=1e-3)
    sim = Simulation(nx, ny, Lambda=1e-3)
    sim.set_fields(**f)
    st = initial_state(f)
    phs = ex.phi_star(st.phi, st.phi_prev)
    Mx, My = ex.mobility_faces(phs, prm.Lambda)
    A = asm.ch_matrix(nx, ny, prm.dt, prm.Gamma1, Mx, My)
    assert _rel(sim.apply_operator("ch", x).ravel(), A @ x.ravel()) <= 1e-13
    bx, by = ex.pressure_faces(st.phi, prm.rho_n, prm.rho_s)
    Ap = asm.poisson_matrix(nx, ny, bx, by)
    assert _rel(sim.apply_operator("poisson", x).ravel(), Ap @ x.ravel()) <= 1e-13
    (Au, _), (Av, _) = momentum_systems(st, phs, prm)
    assert _rel(sim.apply_operator("mom_u", x).ravel(), Au @ x.ravel()) <= 1e-13
    xv = x.copy()
    xv[0] = 0.0
    assert _rel(sim.apply_operator("mom_v", xv).ravel(), Av @ xv.ravel()) <= 1e-13
    sim.close()


def test_variable_density_poisson_operator():
    from paper_1811_11842_b200 import Simulation
    from oracle import assemble as asm, explicit as ex
    from workloads import initial_fields
    nx, ny = 33, 29
    f = initial_fields(nx, ny, seed=3)
    x = np.random.default_rng(5).random((ny, nx))
    sim = Simulation(nx, ny, rho_n=1.7, rho_s=0.9)
    sim.set_fields(**f)
    bx, by = ex.pressure_faces(f["phi"], 1.7, 0.9)
    Ap = asm.poisson_matrix(nx, ny, bx, by)
    assert _rel(sim.apply_operator("poisson", x).ravel(), Ap @ x.ravel()) <= 1e-13
    sim.close()


def test_variable_density_step_matches_oracle():
    got, ref, _, _ = _run_both(40, 32, 1, rho_n=1.5, rho_s=1.0)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (k, _rel(got[k], ref[k]))


def test_device_buffers_roundtrip():
    import torch
    from paper_1811_11842_b200 import Simulation
    from workloads import initial_fields
    f = initial_fields(32, 32, seed=2)
    sim = Simulation(32, 32)
    dev = {k: torch.from_numpy(v).cuda() for k, v in f.items()}
    sim.set_fields(**dev)
    back = sim.get_fields(device=True)
    torch.cuda.synchronize()
    for k in FIELDS:
        assert np.array_equal(back[k].cpu().numpy(), f[k])
    sim.close()


def test_mass_conserved_and_divergence_free_on_gpu():
    from paper_1811_11842_b200 import Simulation
    from oracle import explicit as ex
    from workloads import initial_fields
    f = initial_fields(96, 96, seed=8)
    sim = Simulation(96, 96, eps=0.0)
    sim.set_fields(**f)
    m0 = ex.mass(f["phi"])
    for _ in range(5):
        sim.step(1)
        g = sim.get_fields()
        assert abs(ex.mass(g["phi"]) - m0) / m0 < 1e-12
        d = ex.divergence(g["u"], g["v"])
        assert np.abs(d).max() < 1e-6
    sim.close()


@pytest.mark.parametrize("variant", ["0", "1", "2", "3"])
@pytest.mark.parametrize("nx,ny", [(64, 48), (300, 70)])
def test_cg_kernel_variants_match_oracle(variant, nx, ny, monkeypatch):
    """Two-kernel Hestenes-Stiefel CG: scalar (0), register-pipelined vector (1),
    TMA ring (2); single-reduction fused sweep (3, default), including a ragged
    chunk (nx = 300: 256 + 44 columns)."""
    monkeypatch.setenv("CHB_VEC", variant)
    got, ref, st, iters = _run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (variant, k, _rel(got[k], ref[k]))


@pytest.mark.parametrize("variant,strip", [("1", "3"), ("2", "3"), ("3", "1"), ("3", "2"),
                                           ("3", "3")])
def test_cg_kernel_variants_short_strips(variant, strip, monkeypatch):
    """Forced 1-3-row strips: many strips per slab, halo rows at every strip edge
    (for the fused sweep: redundant z_{i+1} rows at every strip edge)."""
    monkeypatch.setenv("CHB_VEC", variant)
    monkeypatch.setenv("CHB_STRIP", strip)
    got, ref, _, _ = _run_both(64, 40, 1, rtol=1e-12)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (variant, k, _rel(got[k], ref[k]))


@pytest.mark.parametrize("cg3", ["0", "1"])
@pytest.mark.parametrize("nx,ny,strip", [(64, 48, "0"), (300, 70, "0"), (64, 40, "1"),
                                         (64, 40, "2")])
def test_single_reduction_recurrences(cg3, nx, ny, strip, monkeypatch):
    """Single-reduction CG with the three-term z recurrence (1, default: the
    sweep reads z_{i-1}, no s vector) and with the s = A p recurrence (0):
    both match the oracle's Hestenes-Stiefel CG fields and iteration counts,
    on ragged chunks and on 1-2-row strips (halo rows of z_{i-1} at every
    strip edge)."""
    monkeypatch.setenv("CHB_VEC", "3")
    monkeypatch.setenv("CHB_CG3", cg3)
    if strip != "0":
        monkeypatch.setenv("CHB_STRIP", strip)
    got, ref, st, iters = _run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (cg3, k, _rel(got[k], ref[k]))
    for sysname in ("nutrient", "u", "v", "p"):
        assert abs(st["iters_last"][sysname] - iters[-1][sysname]) <= 2, (sysname, st, iters)


def test_skewed_array_starts(monkeypatch):
    """CHB_SKEW: arrays start at staggered offsets inside their allocations
    (DRAM-channel experiment); the step is unchanged."""
    monkeypatch.setenv("CHB_SKEW", "4352")
    got, ref, _, _ = _run_both(64, 48, 1, rtol=1e-12)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (k, _rel(got[k], ref[k]))


# ------------------------------------------------------------ isolated solves
def _solve_case(nx, ny, op, seed=0, **over):
    """GPU ch_solve vs the oracle's textbook Krylov on the assembled matrix,
    same b, same x0, same coefficients (from the seeded state)."""
    from paper_1811_11842_b200 import Simulation, SimParams
    from oracle import assemble as asm, explicit as ex
    from oracle.krylov import bicgstab, cg
    from oracle.step import initial_state, momentum_systems
    from workloads import initial_fields
    f = initial_fields(nx, ny, seed=seed)
    rng = np.random.default_rng(seed + 11)
    b = rng.standard_normal((ny, nx))
    x0 = rng.standard_normal((ny, nx)) * 0.1
    if op == "mom_v":
        b[0] = 0.0
        x0[0] = 0.0
    sp = SimParams(**over)
    prm = _oracle_params(sp)
    sim = Simulation(nx, ny, sp)
    sim.set_fields(**f)
    x = sim.solve(op, b, x0)
    st = sim.stats()
    sim.close()
    s0 = initial_state(f)
    phs = ex.phi_star(s0.phi, s0.phi_prev)
    if op == "poisson":
        bx, by = ex.pressure_faces(s0.phi, prm.rho_n, prm.rho_s)
        A = asm.poisson_matrix(nx, ny, bx, by)
        ref, it = cg(A, b.ravel(), x0.ravel(), 1.0 / A.diagonal(), prm.rtol, prm.maxit,
                     nullspace=True)
        sysname = "p"
    elif op in ("mom_u", "mom_v"):
        (Au, _), (Av, _) = momentum_systems(s0, phs, prm)
        A = Au if op == "mom_u" else Av
        ref, it = cg(A, b.ravel(), x0.ravel(), 1.0 / A.diagonal(), prm.rtol, prm.maxit)
        sysname = "u" if op == "mom_u" else "v"
    else:
        Mx, My = ex.mobility_faces(phs, prm.Lambda)
        A = asm.ch_matrix(nx, ny, prm.dt, prm.Gamma1, Mx, My)
        ref, it = bicgstab(A, b.ravel(), x0.ravel(), 1.0 / A.diagonal(), prm.rtol, prm.maxit)
        sysname = "ch"
    return x, ref.reshape(ny, nx), st["iters_last"][sysname], it


@pytest.mark.parametrize("op", ["poisson", "mom_u", "mom_v", "ch"])
@pytest.mark.parametrize("nx,ny", [(64, 48), (300, 37)])
def test_isolated_solve_matches_oracle(op, nx, ny):
    x, ref, it_gpu, it_ref = _solve_case(nx, ny, op, rtol=1e-12, Lambda=1e-5, rho_n=1.3)
    assert _rel(x, ref) <= 1e-9, (op, _rel(x, ref))
    if op == "ch":
        # BiCGStab's count is not a function of the arithmetic alone: the oracle
        # itself needs 268-306 iterations here when b is perturbed by 1e-15
        assert abs(it_gpu - it_ref) <= 0.35 * it_ref, (it_gpu, it_ref)
    else:
        assert abs(it_gpu - it_ref) <= 2, (it_gpu, it_ref)


def _true_residual_4096(op, kind, variant, monkeypatch, refine=0):
    import torch
    from paper_1811_11842_b200 import Simulation
    from workloads import initial_fields
    monkeypatch.setenv("CHB_VEC", variant)
    n = 4096
    f = initial_fields(n, n, seed=0)
    sim = Simulation(n, n, refine=refine)
    sim.set_fields(**f)
    if kind == "random":
        g = torch.Generator(device="cuda").manual_seed(3)
        b = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    else:   # smooth, large-scale: the spectrum of a step's right-hand sides
        x = (torch.arange(n, dtype=torch.float64, device="cuda") + 0.5) / n
        Y, X = torch.meshgrid(x, x, indexing="ij")
        b = 70.0 * torch.cos(2 * np.pi * X) * torch.cos(np.pi * Y) + 5.0 * torch.sin(6 * np.pi * X)
    if op == "poisson":
        b -= b.mean()
    if op == "mom_v":
        b[0] = 0.0
    xs = sim.solve(op, b.contiguous())
    r = b - sim.apply_operator(op, xs)
    if op == "poisson":
        r -= r.mean()
    st = sim.stats()
    sim.close()
    sysname = {"poisson": "p", "mom_u": "u", "mom_v": "v"}[op]
    return float(torch.linalg.norm(r) / torch.linalg.norm(b)), st["resid_last"][sysname], \
        st["iters_last"][sysname]


@pytest.mark.parametrize("op", ["poisson", "mom_u"])
def test_full_size_solve_true_residual(op, monkeypatch):
    """4096^2 (BASELINE configs[3]) in bench's launch configuration: the
    recursively updated residual the solver stops on must be the true one,
    ||b - A x|| <= 2 rtol ||b|| with A applied by the independent apply kernel
    (broadband right-hand side)."""
    true, rec, _ = _true_residual_4096(op, "random", "3", monkeypatch)
    assert rec <= 1e-10
    assert true <= 2e-10, true


@pytest.mark.parametrize("op", ["poisson", "mom_u"])
def test_full_size_smooth_rhs_residual_gap(op, monkeypatch, record_property):
    """Smooth right-hand side at 4096^2: fp64 CG's recursively updated residual
    drifts from the true one (attainable accuracy ~ eps * kappa, kappa(A_p) ~
    7e6).  The single-reduction sweep must not be worse than the
    Hestenes-Stiefel iteration (same arithmetic class), and both stay below 1e-7."""
    res = {}
    for variant in ("2", "3"):
        res[variant] = _true_residual_4096(op, "smooth", variant, monkeypatch)
        record_property(f"true_resid_v{variant}", res[variant][0])
    print("true residuals (HS, CG-CG):", res)
    assert res["3"][0] <= 3.0 * res["2"][0] + 1e-10, res
    assert res["3"][0] <= 1e-7, res


def test_full_size_operator_samples_match_oracle():
    """4096^2 operator applies on sampled cells (walls, periodic seam, chunk and
    strip edges, random interior) vs the oracle's single-cell brute force."""
    from paper_1811_11842_b200 import Simulation
    from oracle import brute
    from workloads import initial_fields
    n = 4096
    f = initial_fields(n, n, seed=5)
    rng = np.random.default_rng(9)
    x = rng.random((n, n))
    rho_n, rho_s = 1.4, 0.8
    sim = Simulation(n, n, rho_n=rho_n, rho_s=rho_s, Lambda=1e-5)
    sim.set_fields(**f)
    yp = sim.apply_operator("poisson", x)
    yc = sim.apply_operator("ch", x)
    sim.close()
    cells = [(0, 0), (0, n - 1), (n - 1, 0), (n - 1, n - 1), (1, 255), (1, 256), (2047, 4095),
             (n - 2, 3840), (228, 511), (229, 512)]
    cells += [tuple(v) for v in rng.integers(0, n, size=(30, 2))]
    for j, i in cells:
        rp = brute.poisson_at(f["phi"], x, j, i, rho_n, rho_s)
        assert abs(yp[j, i] - rp) <= 1e-12 * max(1.0, abs(rp)) * 1e3, (j, i, yp[j, i], rp)
        rc = brute.ch_apply_at(f["phi"], x, j, i, 1e-4, 33.467, 1e-5)
        assert abs(yc[j, i] - rc) <= 1e-11 * max(1.0, abs(rc)) * 1e3, (j, i, yc[j, i], rc)


def test_full_size_step_invariants():
    """One 4096^2 step (bench workload): every solve reaches rtol, the new
    velocity is discretely divergence free to solver accuracy, and with the
    growth term off the phi mass is conserved (telescoping fluxes)."""
    from paper_1811_11842_b200 import Simulation
    from oracle import explicit as ex
    from workloads import initial_fields
    n = 4096
    f = initial_fields(n, n, seed=0)
    sim = Simulation(n, n, eps=0.0)
    sim.set_fields(**f)
    sim.step(1)
    g = sim.get_fields(("phi", "u", "v", "p"))
    st = sim.stats()
    ap = sim.apply_operator("poisson", g["p"])   # -D beta G p at phi^{n+1}
    sim.close()
    for k, r in st["resid_last"].items():
        assert r <= 1e-10, (k, r)
    m0 = ex.mass(f["phi"])
    assert abs(ex.mass(g["phi"]) - m0) / m0 < 1e-11
    # D_h u^{n+1} = D_h u* - A_p p is the pressure solve's residual, and
    # D_h u* = D_h u^{n+1} + A_p p is its right-hand side (mean-free)
    d = ex.divergence(g["u"], g["v"])
    rhs = d + ap
    rhs -= rhs.mean()
    # = the pressure solve's TRUE residual, which at 4096^2 sits at fp64 CG's
    # attainable accuracy (see test_full_size_smooth_rhs_residual_gap)
    assert np.linalg.norm(d - d.mean()) <= 1e-7 * np.linalg.norm(rhs)


@pytest.mark.parametrize("defer", ["2", "5", "8", "12"])
@pytest.mark.parametrize("nx,ny", [(64, 48), (300, 70)])
def test_deferred_px_block_lengths(defer, nx, ny, monkeypatch):
    """Single-reduction CG with p/x updated in the sweep (0) or deferred over
    blocks of m stored z's (2..12): full and partial final blocks."""
    monkeypatch.setenv("CHB_VEC", "3")
    monkeypatch.setenv("CHB_DEFER", defer)
    got, ref, st, iters = _run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (defer, k, _rel(got[k], ref[k]))
    for sysname in ("nutrient", "u", "v", "p"):
        assert abs(st["iters_last"][sysname] - iters[-1][sysname]) <= 2, (sysname, st, iters)


@pytest.mark.parametrize("defer", ["2", "7"])
@pytest.mark.parametrize("op", ["poisson", "mom_v"])
def test_isolated_solve_deferred_modes(defer, op, monkeypatch):
    monkeypatch.setenv("CHB_DEFER", defer)
    x, ref, it_gpu, it_ref = _solve_case(128, 96, op, rtol=1e-12, rho_n=0.7)
    assert _rel(x, ref) <= 1e-9, (op, _rel(x, ref))
    assert abs(it_gpu - it_ref) <= 2, (it_gpu, it_ref)


@pytest.mark.parametrize("nx,ny", [(64, 48), (300, 70), (520, 33)])
def test_persistent_cg_matches_oracle(nx, ny, monkeypatch):
    """Whole CG solves as one cooperative launch (grid barrier + last-CTA
    finalize per iteration, in-kernel p/x blocks): same fields and iteration
    counts as the oracle."""
    monkeypatch.setenv("CHB_PERSIST", "1")
    got, ref, st, iters = _run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (k, _rel(got[k], ref[k]))
    for sysname in ("nutrient", "u", "v", "p"):
        assert abs(st["iters_last"][sysname] - iters[-1][sysname]) <= 2, (sysname, st, iters)


@pytest.mark.parametrize("op", ["poisson", "mom_v"])
def test_persistent_isolated_solve(op, monkeypatch):
    monkeypatch.setenv("CHB_PERSIST", "1")
    monkeypatch.setenv("CHB_DEFER", "5")
    x, ref, it_gpu, it_ref = _solve_case(128, 96, op, rtol=1e-12, rho_n=0.7)
    assert _rel(x, ref) <= 1e-9, (op, _rel(x, ref))
    assert abs(it_gpu - it_ref) <= 2, (it_gpu, it_ref)


def test_config2_1024_steps_invariants():
    """BASELINE.json configs[2] (1024^2, here 5 of its 50 steps): every solve
    reaches rtol, the projected velocity is divergence free to the pressure
    solve's accuracy, and with growth off phi's mass is conserved."""
    from paper_1811_11842_b200 import Simulation
    from oracle import explicit as ex
    from workloads import initial_fields
    n = 1024
    f = initial_fields(n, n, seed=0)
    sim = Simulation(n, n, eps=0.0)
    sim.set_fields(**f)
    m0 = ex.mass(f["phi"])
    for _ in range(5):
        sim.step(1)
        st = sim.stats()
        for k, r in st["resid_last"].items():
            assert r <= 1e-10, (k, r)
    g = sim.get_fields(("phi", "u", "v", "p"))
    ap = sim.apply_operator("poisson", g["p"])
    sim.close()
    assert abs(ex.mass(g["phi"]) - m0) / m0 < 1e-11
    d = ex.divergence(g["u"], g["v"])
    rhs = d + ap
    rhs -= rhs.mean()
    assert np.linalg.norm(d - d.mean()) <= 1e-8 * np.linalg.norm(rhs)


@pytest.mark.parametrize("defer", ["4", "8", "32"])
@pytest.mark.parametrize("nx,ny", [(64, 48), (300, 70)])
def test_async_px_matches_oracle(defer, nx, ny, monkeypatch):
    """p/x block updates on a side stream overlapped with the sweeps (the main
    stream waits for block b before the finalize that reuses its coefficient
    table): same fields and iteration counts as the oracle."""
    monkeypatch.setenv("CHB_PXASYNC", "1")
    monkeypatch.setenv("CHB_DEFER", defer)
    got, ref, st, iters = _run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (defer, k, _rel(got[k], ref[k]))
    for sysname in ("nutrient", "u", "v", "p"):
        assert abs(st["iters_last"][sysname] - iters[-1][sysname]) <= 2, (sysname, st, iters)


@pytest.mark.parametrize("nx,ny", [(45, 38), (33, 21), (8, 6), (6, 4), (4, 4)])
def test_odd_and_tiny_grids_match_oracle(nx, ny):
    """Odd nx (two-kernel CG and tile CH apply fallback) and the smallest grids
    the library accepts (single chunk, strips of one or two rows)."""
    got, ref, st, iters = _run_both(nx, ny, 1, rtol=1e-12, Lambda=1e-5)
    for k in FIELDS:
        assert _rel(got[k], ref[k]) <= 1e-9, (nx, ny, k, _rel(got[k], ref[k]))



@pytest.mark.parametrize("op", ["poisson", "mom_u"])
def test_full_size_true_residual_refinement(op, monkeypatch, record_property):
    """params.refine: restarting CG from the converged x until its own
    initialisation (b - A x from scratch) already meets rtol drives the TRUE
    residual to rtol at 4096^2 even for a smooth right-hand side."""
    base = _true_residual_4096(op, "smooth", "3", monkeypatch)
    ref = _true_residual_4096(op, "smooth", "3", monkeypatch, refine=4)
    record_property("iters_base", base[2])
    record_property("iters_refined", ref[2])
    print("true residual, iterations: plain", base, "refined", ref)
    assert ref[0] <= 2e-10, ref
    assert ref[2] >= base[2]
