"""BASELINE.json configs[4], second part: isolated matvec sweeps of the
Cahn-Hilliard (13-point, with its advection part) and pressure-Poisson
(5-point) stencils on random fp64 fields uniform in [0, 1), device-resident.
The time per apply is the library's own CUDA-event timing of the stencil
launch on its stream (coefficient set-up and copies excluded); bytes are
algorithmic (CH: read x, phi*, u, v, write y = 40 B/cell; Poisson: read x,
write y = 16 B/cell)."""
from __future__ import annotations

BYTES = {"ch": 40.0, "poisson": 16.0}


def sweep(sizes=(1024, 4096, 16384), reps=20, peak_gbs=None):
    import torch
    from . import Simulation
    out = []
    for n in sizes:
        g = torch.Generator(device="cuda").manual_seed(n)
        phi = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
        sim = Simulation(n, n, Lambda=1e-5)
        sim.set_stream(torch.cuda.current_stream())
        sim.set_fields(phi=phi.contiguous())
        sim.time_index = 10           # Crank-Nicolson weights (past the start-up steps)
        x = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
        for op in ("ch", "poisson"):
            sim.apply_operator(op, x)  # warm-up
            sim.reset_stats()
            sim.enable_timing(1)
            for _ in range(reps):
                sim.apply_operator(op, x)
            st = sim.stats()
            sim.enable_timing(0)
            kc = st["kernels"]["ch_apply" if op == "ch" else "op_apply"]
            ms = kc["ms"] / max(kc["timed"], 1)
            gbs = BYTES[op] * n * n / (ms * 1e-3) / 1e9 if ms > 0 else None
            rec = {"op": op, "n": n, "ms_per_apply": ms, "GBps": gbs, "bytes_per_cell": BYTES[op]}
            if peak_gbs and gbs:
                rec["frac"] = gbs / peak_gbs
            out.append(rec)
        sim.close()
        del phi, x
        torch.cuda.empty_cache()
    return out
