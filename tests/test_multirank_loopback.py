"""The library's MULTI-RANK code path (nranks > 1: rank-local slabs, halo rows
and partial-sum allgathers through the NCCL API, cross-rank finalize) run with
2-3 ranks as host threads of one process on one GPU, through an in-process
loopback stand-in for libnccl.so.2 (tests/fake_nccl/fake_nccl.cpp, loaded via
CHB_NCCL_LIB).  The fields must equal a single-rank run's up to rounding of the
reduction order (same bar as the virtual-slab tests).  The real NCCL transport
is the same calls into the real library; this run checks the rank / row /
ordering logic above it without a second GPU."""
import os
import subprocess
import threading

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE_SRC = os.path.join(ROOT, "tests", "fake_nccl", "fake_nccl.cpp")
FAKE_LIB = os.path.join(ROOT, "tests", "fake_nccl", "libfake_nccl.so")
FIELDS = ("phi", "c", "u", "v", "p")


def _build_fake():
    if os.path.exists(FAKE_LIB) and os.path.getmtime(FAKE_LIB) >= os.path.getmtime(FAKE_SRC):
        return FAKE_LIB
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(cuda, "include"),
                    FAKE_SRC, "-o", FAKE_LIB, "-L", os.path.join(cuda, "lib64"), "-lcudart"],
                   check=True, capture_output=True)
    return FAKE_LIB


def test_fake_transport_builds():
    """The loopback stand-in compiles (host C++ against the CUDA runtime)."""
    assert os.path.exists(_build_fake())


def _run_ranks(nx, ny, nranks, steps, vslabs=1, **kw):
    import torch
    from paper_1811_11842_b200 import Simulation, unique_id
    from workloads import initial_fields
    uid = unique_id()
    out, its, errs, modes = [None] * nranks, [None] * nranks, [], [None] * nranks
    sims = [Simulation(nx, ny, rank=r, nranks=nranks, device=0, virtual_slabs=vslabs, **kw)
            for r in range(nranks)]

    def run(r):
        try:
            sim = sims[r]
            sim.set_stream(torch.cuda.Stream())
            sim.comm_init(uid)
            modes[r] = sim.comm_mode
            rows = (sim.row0, sim.row0 + sim.nrows)
            sim.set_fields(**initial_fields(nx, ny, seed=4, rows=rows))
            sim.step(steps)
            out[r] = (rows, sim.get_fields())
            its[r] = sim.stats()["iters_last"]
        except Exception as e:  # surfaced in the main thread
            errs.append((r, repr(e)))

    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "rank thread hung (transport deadlock)"
    for s in sims:
        s.close()
    assert not errs, errs
    # ranks sharing one GPU never use the peer-memory sweep (their kernels
    # would wait on one another): the NCCL transport carries the iteration
    assert modes == ["nccl"] * nranks, modes
    glob = {k: np.zeros((ny, nx)) for k in FIELDS}
    for (r0, r1), f in out:
        for k in FIELDS:
            glob[k][r0:r1] = f[k]
    return glob, its


@pytest.mark.gpu
@pytest.mark.parametrize("nranks,solver,vslabs", [(2, "bicgstab", 1), (3, "bicgstab", 1),
                                                  (2, "gmres", 1), (2, "bicgstab", 2)])
def test_multirank_loopback_matches_single_rank(nranks, solver, vslabs, monkeypatch):
    monkeypatch.setenv("CHB_NCCL_LIB", _build_fake())
    from paper_1811_11842_b200 import Simulation
    from workloads import initial_fields
    nx, ny = 40, 36
    kw = dict(Lambda=1e-5, rtol=1e-13, ch_solver=solver)
    glob, its = _run_ranks(nx, ny, nranks, 2, vslabs=vslabs, **kw)
    sim = Simulation(nx, ny, **kw)
    sim.set_fields(**initial_fields(nx, ny, seed=4))
    sim.step(2)
    ref = sim.get_fields()
    it1 = sim.stats()["iters_last"]
    sim.close()
    for k in FIELDS:
        rel = np.linalg.norm(glob[k] - ref[k]) / max(np.linalg.norm(ref[k]), 1e-300)
        tol = 1e-10 if k == "v" else 1e-11  # as the virtual-slab tests (R17)
        assert rel <= tol, (k, rel)
    for r in range(nranks):
        assert its[r] == its[0], its  # every rank runs the same global iteration
    for k in it1:
        assert abs(its[0][k] - it1[k]) <= 3 + 0.1 * it1[k], (its[0], it1)
