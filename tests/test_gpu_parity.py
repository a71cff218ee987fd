"""GPU path (C ABI, sm_100a kernels) vs the CPU oracle, element by element.

Tolerances (north_star): relative L2 <= 1e-9 per field after one step; every
Krylov solve reaches ||r||/||b|| <= 1e-10.  Operator applies are exact up to
rounding: relative L2 <= 1e-13.  Long trajectories and full-size (4096^2)
checks: tests/test_gpu_fullsize.py; oracle goldens: tests/test_gpu_goldens.py.
"""
import numpy as np
import pytest

from gpu_helpers import FIELDS, oracle_params, rel, run_both, stream_velocity

pytestmark = pytest.mark.gpu


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
        a, _ = step(a, oracle_params(sp))
        b, _ = step(b, oracle_params(sp, rtol=1e-13))
    return {k: rel(getattr(a, k), getattr(b, k)) for k in FIELDS}


@pytest.mark.parametrize("nx,ny", [(64, 64), (50, 37), (130, 70)])
def test_one_step_matches_oracle(nx, ny):
    """Element-by-element parity, north_star bound 1e-9 on every field.  The
    solves run to rtol 1e-12 on both sides (<= north_star's 1e-10, R17)."""
    got, ref, st, iters = run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS + ("u_star", "v_star"):
        assert rel(got[k], ref[k]) <= 1e-9, (k, rel(got[k], ref[k]))
    for sysname, n in iters[-1].items():
        assert abs(st["iters_last"][sysname] - n) <= 2, (sysname, st["iters_last"], iters[-1])
        assert st["resid_last"][sysname] <= 1e-12


def test_three_steps_carry_the_momentum_guess():
    """R25: the momentum solves of step n start from u*, v* of step n - 1 on
    both sides -- equal iteration counts (a solve started from u^n instead
    needs measurably more) and every field, u* and v* included, within 1e-9."""
    got, ref, st, iters = run_both(64, 64, 3, rtol=1e-12)
    for k in FIELDS + ("u_star", "v_star"):
        assert rel(got[k], ref[k]) <= 1e-9, (k, rel(got[k], ref[k]))
    for sysname, n in iters[-1].items():
        assert abs(st["iters_last"][sysname] - n) <= 2, (sysname, st["iters_last"], iters[-1])


def test_restart_from_saved_state_is_bitwise():
    """Checkpoint / resume: the state (fields, phi^{n-1}, u*, v*, time index)
    read out after 2 steps and set into a fresh handle gives bit-for-bit the
    third step of an uninterrupted run."""
    from paper_1811_11842_b200 import Simulation
    from workloads import initial_fields
    names = FIELDS + ("phi_prev", "u_star", "v_star")
    n = 64
    f = initial_fields(n, n, seed=2)
    a = Simulation(n, n)
    a.set_fields(**f)
    a.step(2)
    saved = a.get_fields(names)
    tidx = a.time_index
    a.step(1)
    ref = a.get_fields(names)
    a.close()
    b = Simulation(n, n)
    b.set_fields(**{k: saved[k] for k in FIELDS})
    for k in ("phi_prev", "u_star", "v_star"):
        b.set_field(k, saved[k])
    b.time_index = tidx
    b.step(1)
    got = b.get_fields(names)
    b.close()
    for k in names:
        assert np.array_equal(got[k], ref[k]), k


@pytest.mark.parametrize("refine", [0, 2])
@pytest.mark.parametrize("nx,ny", [(64, 64), (130, 70)])
def test_one_step_at_north_star_rtol(nx, ny, refine):
    """At north_star's rtol 1e-10 every field matches within 1e-9 plus the
    oracle's own stopping-point sensitivity (R17), iteration counts agree
    within 2 (+ the restart iterations of the true-residual refinement, R21)
    and every solve reaches 1e-10."""
    got, ref, st, iters = run_both(nx, ny, 1, refine=refine)
    tr = _oracle_truncation(nx, ny)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9 + tr[k], (k, rel(got[k], ref[k]), tr[k])
    for sysname, n in iters[-1].items():
        slack = 2 + (8 if refine and sysname != "ch" else 0)
        assert -2 <= st["iters_last"][sysname] - n <= slack, (sysname, st["iters_last"], iters[-1])
        assert st["resid_last"][sysname] <= 1e-10


def test_moving_fluid_steps_match_oracle():
    """A state with a divergence-free velocity field and a tilted phi, so that
    every term is live from the first step: the implicit CN advection inside
    the CH system (R12), the convection and the viscous transpose part of R
    (R6), the volume-fraction clip (R24, phi dips below 0), the start-up step
    (startup_be = 1, R23) and then CN steps."""
    nx, ny = 96, 64
    from workloads import initial_fields
    f = initial_fields(nx, ny, seed=3)
    u, v = stream_velocity(nx, ny, seed=4, scale=0.02)
    f["u"], f["v"] = u, v
    f["phi"] = f["phi"] - 0.002
    got, ref, st, iters = run_both(nx, ny, 3, fields=f, rtol=1e-12, startup_be=1, Lambda=1e-6)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (k, rel(got[k], ref[k]))
    assert min(got["phi"].min(), f["phi"].min()) < 0


def test_crank_nicolson_viscous_and_explicit_advection_variants():
    """theta_visc = 1/2 (Crank-Nicolson viscous term) and theta_adv = 0
    (explicit advection) follow the oracle too (the weights are parameters)."""
    nx, ny = 64, 48
    from workloads import initial_fields
    f = initial_fields(nx, ny, seed=5)
    u, v = stream_velocity(nx, ny, seed=6, scale=0.01)
    f["u"], f["v"] = u, v
    got, ref, _, _ = run_both(nx, ny, 2, fields=f, rtol=1e-12, theta_visc=0.5, theta_adv=0.0,
                              theta_ch=0.75)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (k, rel(got[k], ref[k]))


def test_one_step_gmres_matches_oracle():
    got, ref, st, _ = run_both(64, 64, 1, ch_solver="gmres", Lambda=1e-5)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (k, rel(got[k], ref[k]))


def test_bicgstab_nontrivial_ch_system():
    """Lambda large enough that the CH system is far from I/dt (many iterations)."""
    got, ref, st, iters = run_both(48, 40, 2, Lambda=1e-5)
    assert st["iters_last"]["ch"] >= 5
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (k, rel(got[k], ref[k]))


@pytest.mark.parametrize("nx,ny", [(46, 38), (34, 21), (8, 6), (6, 4), (4, 4)])
def test_small_and_ragged_grids_match_oracle(nx, ny):
    """Ragged chunks and the smallest grids the library accepts (single chunk,
    strips of one or two rows)."""
    got, ref, st, iters = run_both(nx, ny, 1, rtol=1e-12, Lambda=1e-5)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (nx, ny, k, rel(got[k], ref[k]))


def test_odd_nx_rejected():
    from paper_1811_11842_b200 import CHError, Simulation
    with pytest.raises(CHError):
        Simulation(45, 38)


@pytest.mark.parametrize("ms", ["1", "0"])
@pytest.mark.parametrize("cg3", ["1", "0"])
@pytest.mark.parametrize("slabs", [2, 3])
def test_virtual_slabs_match_single_slab(slabs, cg3, ms, monkeypatch):
    """Slab decomposition in y with halo exchange reproduces the 1-slab step
    (CG: three-term z recurrence, z halos only; and s recurrence, z + s
    halos), with the CG iteration as ONE launch over all slabs (ms = 1: the
    sweep stores its slab-edge rows into the neighbours' ghost rows and the
    last slab combines the partial sums) or as per-slab launches + halo copies
    + a finalize kernel (ms = 0, the multi-rank code path).  Dot products sum
    in a different order per decomposition, so the solves run to rtol 1e-13
    (differences are rounding propagated through the CG iterations)."""
    from paper_1811_11842_b200 import Simulation
    from workloads import initial_fields
    monkeypatch.setenv("CHB_CG3", cg3)
    monkeypatch.setenv("CHB_MS", ms)
    f = initial_fields(40, 36, seed=4)
    u, v = stream_velocity(40, 36, seed=2, scale=0.01)
    f["u"], f["v"] = u, v
    out, its = [], []
    for s in (1, slabs):
        sim = Simulation(40, 36, virtual_slabs=s, Lambda=1e-5, rtol=1e-13)
        sim.set_fields(**f)
        sim.step(2)
        out.append(sim.get_fields())
        its.append(sim.stats()["iters_last"])
        sim.close()
    for k in FIELDS:
        tol = 1e-10 if k == "v" else 1e-11
        assert rel(out[1][k], out[0][k]) <= tol, (k, rel(out[1][k], out[0][k]))
    for k in its[0]:
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
        assert rel(out[1][k], out[0][k]) <= tol, (k, rel(out[1][k], out[0][k]))


def test_operator_applies_match_assembled_matrices():
    """The four isolated applies vs the oracle's assembled matrices on a state
    with a moving fluid (the CH operator's advection part is live)."""
    from paper_1811_11842_b200 import Simulation
    from oracle import assemble as asm, explicit as ex
    from oracle.step import initial_state, momentum_systems
    from workloads import initial_fields
    nx, ny = 46, 38
    f = initial_fields(nx, ny, seed=1)
    f["u"], f["v"] = stream_velocity(nx, ny, seed=7, scale=0.05)
    x = np.random.default_rng(0).random((ny, nx))
    sim = Simulation(nx, ny, Lambda=1e-3)
    prm = oracle_params(sim.params)
    sim.set_fields(**f)
    sim.time_index = 10      # past the backward-Euler start-up: CN weights (R23)
    st = initial_state(f)
    phs = ex.phi_star(st.phi, st.phi_prev)
    Mx, My = ex.mobility_faces(phs, prm.Lambda)
    A = asm.ch_matrix(nx, ny, prm.dt, prm.Gamma1, Mx, My, prm.theta_ch, prm.theta_adv, st.u, st.v)
    assert rel(sim.apply_operator("ch", x).ravel(), A @ x.ravel()) <= 1e-13
    bx, by = ex.pressure_faces(st.phi, prm.rho_n, prm.rho_s)
    Ap = asm.poisson_matrix(nx, ny, bx, by)
    assert rel(sim.apply_operator("poisson", x).ravel(), Ap @ x.ravel()) <= 1e-13
    (Au, _), (Av, _) = momentum_systems(st, phs, prm)
    assert rel(sim.apply_operator("mom_u", x).ravel(), Au @ x.ravel()) <= 1e-13
    xv = x.copy()
    xv[0] = 0.0
    assert rel(sim.apply_operator("mom_v", xv).ravel(), Av @ xv.ravel()) <= 1e-13
    from oracle.step import nutrient_system
    An, _ = nutrient_system(st, st.phi, prm)
    assert rel(sim.apply_operator("nutrient", x).ravel(), An @ x.ravel()) <= 1e-13
    sim.close()


def test_variable_density_poisson_operator():
    from paper_1811_11842_b200 import Simulation
    from oracle import assemble as asm, explicit as ex
    from workloads import initial_fields
    nx, ny = 34, 29
    f = initial_fields(nx, ny, seed=3)
    x = np.random.default_rng(5).random((ny, nx))
    sim = Simulation(nx, ny, rho_n=1.7, rho_s=0.9)
    sim.set_fields(**f)
    bx, by = ex.pressure_faces(f["phi"], 1.7, 0.9)
    Ap = asm.poisson_matrix(nx, ny, bx, by)
    assert rel(sim.apply_operator("poisson", x).ravel(), Ap @ x.ravel()) <= 1e-13
    sim.close()


def test_variable_density_step_matches_oracle():
    got, ref, _, _ = run_both(40, 32, 1, rho_n=1.5, rho_s=1.0, rtol=1e-12)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (k, rel(got[k], ref[k]))


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
    assert sim.time_index == 0
    sim.step(1)
    assert sim.time_index == 1
    sim.time_index = 7
    assert sim.time_index == 7
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


# ----------------------------------------- production launch geometry (strips)
@pytest.mark.parametrize("slabs", [3])
@pytest.mark.parametrize("strip", ["2", "12"])
def test_virtual_slabs_forced_strips(strip, slabs, monkeypatch):
    """One-launch multi-slab sweep with forced strip heights (slab-edge rows
    inside and at the ends of strips) on a ragged 300 x 200 grid, all operator
    kinds, against the oracle."""
    from workloads import initial_fields
    monkeypatch.setenv("CHB_STRIP", strip)
    nx, ny = 300, 200
    f = initial_fields(nx, ny, seed=9)
    f["u"], f["v"] = stream_velocity(nx, ny, seed=9, scale=0.01)
    got, ref, st, iters = run_both(nx, ny, 2, slabs=slabs, fields=f, rtol=1e-12, rho_n=1.2,
                                   Lambda=1e-6)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (strip, k, rel(got[k], ref[k]))


@pytest.mark.parametrize("strip", ["1", "2", "3", "12", "40"])
def test_forced_strips_all_operator_kinds(strip, monkeypatch):
    """Forced strip heights at ~300 x 200 (two column chunks, one ragged): the
    sweeps' shared-memory rings wrap (strip > ring depth: mbarrier phase flips,
    slot refills), the two-row pair() path runs, and every strip edge has
    redundant halo rows -- for all five CG operator kinds (Poisson const/var,
    nutrient, momentum u/v) and the CH apply.  Two steps with a moving fluid."""
    from workloads import initial_fields
    monkeypatch.setenv("CHB_STRIP", strip)
    nx, ny = 300, 200
    f = initial_fields(nx, ny, seed=9)
    f["u"], f["v"] = stream_velocity(nx, ny, seed=9, scale=0.01)
    got, ref, st, iters = run_both(nx, ny, 2, fields=f, rtol=1e-12, rho_n=1.2, Lambda=1e-6)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (strip, k, rel(got[k], ref[k]))
    for sysname in ("nutrient", "u", "v", "p"):
        assert abs(st["iters_last"][sysname] - iters[-1][sysname]) <= 2, (sysname, st, iters)


@pytest.mark.parametrize("cg3", ["0", "1"])
@pytest.mark.parametrize("nx,ny,strip", [(64, 48, "0"), (300, 70, "0"), (64, 40, "1"),
                                         (64, 40, "2")])
def test_single_reduction_recurrences(cg3, nx, ny, strip, monkeypatch):
    """Single-reduction CG with the three-term z recurrence (1, default) and
    the s = A p recurrence (0): both match the oracle's Hestenes-Stiefel CG
    fields and iteration counts (R18, R22)."""
    monkeypatch.setenv("CHB_CG3", cg3)
    if strip != "0":
        monkeypatch.setenv("CHB_STRIP", strip)
    got, ref, st, iters = run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (cg3, k, rel(got[k], ref[k]))
    for sysname in ("nutrient", "u", "v", "p"):
        assert abs(st["iters_last"][sysname] - iters[-1][sysname]) <= 2, (sysname, st, iters)


@pytest.mark.parametrize("defer", ["2", "5", "8", "12"])
@pytest.mark.parametrize("nx,ny", [(64, 48), (300, 70)])
def test_deferred_px_block_lengths(defer, nx, ny, monkeypatch):
    """p/x deferred over blocks of m stored z's (2..12): full and partial final blocks."""
    monkeypatch.setenv("CHB_DEFER", defer)
    got, ref, st, iters = run_both(nx, ny, 1, rtol=1e-12)
    for k in FIELDS:
        assert rel(got[k], ref[k]) <= 1e-9, (defer, k, rel(got[k], ref[k]))
    for sysname in ("nutrient", "u", "v", "p"):
        assert abs(st["iters_last"][sysname] - iters[-1][sysname]) <= 2, (sysname, st, iters)


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
    f["u"], f["v"] = stream_velocity(nx, ny, seed=seed + 1, scale=0.02)
    rng = np.random.default_rng(seed + 11)
    b = rng.standard_normal((ny, nx))
    x0 = rng.standard_normal((ny, nx)) * 0.1
    if op == "mom_v":
        b[0] = 0.0
        x0[0] = 0.0
    sp = SimParams(**over)
    prm = oracle_params(sp)
    sim = Simulation(nx, ny, sp)
    sim.set_fields(**f)
    sim.time_index = 10      # past the backward-Euler start-up: CN weights (R23)
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
    elif op == "nutrient":
        from oracle.step import nutrient_system
        A, _ = nutrient_system(s0, s0.phi, prm)
        ref, it = cg(A, b.ravel(), x0.ravel(), 1.0 / A.diagonal(), prm.rtol, prm.maxit)
        sysname = "nutrient"
    else:
        Mx, My = ex.mobility_faces(phs, prm.Lambda)
        A = asm.ch_matrix(nx, ny, prm.dt, prm.Gamma1, Mx, My, prm.theta_ch, prm.theta_adv,
                          s0.u, s0.v)
        ref, it = bicgstab(A, b.ravel(), x0.ravel(), 1.0 / A.diagonal(), prm.rtol, prm.maxit)
        sysname = "ch"
    return x, ref.reshape(ny, nx), st["iters_last"][sysname], it


def _momentum_matrix(op, nx, ny, seed=0, **over):
    from paper_1811_11842_b200 import SimParams
    from oracle import explicit as ex
    from oracle.step import initial_state, momentum_systems
    from workloads import initial_fields
    f = initial_fields(nx, ny, seed=seed)
    s0 = initial_state(f)
    (Au, _), (Av, _) = momentum_systems(s0, ex.phi_star(s0.phi, s0.phi_prev),
                                        oracle_params(SimParams(**over)))
    return Au if op == "mom_u" else Av


def _check_momentum_solve(op, nx, ny, x, ref, it_gpu, it_ref, seed=0, **over):
    """The momentum operators carry the viscosity contrast eta(0.3)/eta(0) ~ 1e5
    (R6): for a random b, neither fp64 CG attains a TRUE residual near rtol
    (attainable accuracy ~ eps kappa).  The GPU solve must match the textbook
    CG's own true residual (same iterates in exact arithmetic, rounding order
    differs) and its iteration count."""
    A = _momentum_matrix(op, nx, ny, seed, **over)
    b = np.random.default_rng(seed + 11).standard_normal((ny, nx))
    if op == "mom_v":
        b[0] = 0.0
    bn = np.linalg.norm(b)
    t_gpu = np.linalg.norm(b.ravel() - A @ x.ravel()) / bn
    t_ref = np.linalg.norm(b.ravel() - A @ ref.ravel()) / bn
    assert t_gpu <= max(2e-12, 10.0 * t_ref), (op, t_gpu, t_ref)
    assert rel(x, ref) <= 1e-5, (op, rel(x, ref))
    # rtol 1e-12 sits near this system's attainable accuracy: the last iterations are
    # rounding-order dependent
    assert abs(it_gpu - it_ref) <= 2 + 0.05 * it_ref, (it_gpu, it_ref)


@pytest.mark.parametrize("op", ["poisson", "mom_u", "mom_v", "ch", "nutrient"])
@pytest.mark.parametrize("nx,ny", [(64, 48), (300, 37)])
def test_isolated_solve_matches_oracle(op, nx, ny):
    """Same b, x0 and coefficients on both sides (see _check_momentum_solve for
    the momentum operators)."""
    over = dict(rtol=1e-12, Lambda=1e-5, rho_n=1.3)
    x, ref, it_gpu, it_ref = _solve_case(nx, ny, op, **over)
    if op in ("mom_u", "mom_v"):
        _check_momentum_solve(op, nx, ny, x, ref, it_gpu, it_ref, **over)
        return
    assert rel(x, ref) <= 1e-9, (op, rel(x, ref))
    if op == "ch":
        # BiCGStab's count is not a function of the arithmetic alone (the
        # oracle itself moves by tens of iterations when b is perturbed by 1e-15)
        assert abs(it_gpu - it_ref) <= 0.35 * it_ref + 2, (it_gpu, it_ref)
    else:
        assert abs(it_gpu - it_ref) <= 2, (it_gpu, it_ref)


@pytest.mark.parametrize("defer", ["2", "7"])
@pytest.mark.parametrize("op", ["poisson", "mom_v"])
def test_isolated_solve_deferred_modes(defer, op, monkeypatch):
    monkeypatch.setenv("CHB_DEFER", defer)
    x, ref, it_gpu, it_ref = _solve_case(128, 96, op, rtol=1e-12, rho_n=0.7)
    if op == "mom_v":
        _check_momentum_solve(op, 128, 96, x, ref, it_gpu, it_ref, rtol=1e-12, rho_n=0.7)
    else:
        assert rel(x, ref) <= 1e-9, (op, rel(x, ref))
        assert abs(it_gpu - it_ref) <= 2, (it_gpu, it_ref)


def test_not_converged_is_reported_with_the_system_and_residual():
    """A solve hitting maxit raises CH_ERR_NOT_CONVERGED naming the system, the
    iteration count and the residual reached; the state stays at the last
    completed step (here: the initial condition)."""
    from paper_1811_11842_b200 import CHError, Simulation
    from workloads import initial_fields
    f = initial_fields(64, 64, seed=1)
    sim = Simulation(64, 64, maxit=5)
    sim.set_fields(**f)
    with pytest.raises(CHError) as ei:
        sim.step(1)
    msg = str(ei.value)
    assert ei.value.code == 3 and "not converged in 5 iterations" in msg, msg
    assert sim.time_index == 0
    for k in FIELDS:
        assert np.array_equal(sim.get_field(k), f[k]), k
    # a pressure solve that fails leaves p^n as well (the CH, nutrient and
    # momentum solves are cheap at 64^2 with maxit high enough for them)
    sim.close()
    sim = Simulation(64, 64, maxit=100)
    sim.set_fields(**f)
    with pytest.raises(CHError) as ei:
        sim.step(1)
    assert "pressure" in str(ei.value) or "momentum" in str(ei.value), str(ei.value)
    for k in FIELDS:
        assert np.array_equal(sim.get_field(k), f[k]), k
    sim.close()
