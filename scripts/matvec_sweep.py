"""BASELINE.json configs[4], second part: isolated matvec sweeps of the
Cahn-Hilliard (13-point) and pressure-Poisson (5-point) stencils on random
fp64 fields uniform in [0, 1), grids 256^2 .. 16384^2, device-resident.

    python scripts/matvec_sweep.py [--sizes 256 1024 4096 16384] [--reps 20]
One JSON line per (operator, size): time per apply (CUDA events, inputs larger
than L2 from 4096^2 up) and algorithmic GB/s (CH: read x, phi*, write y;
Poisson: read x, write y -- 24 and 16 B/cell).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1811_11842_b200 import Simulation  # noqa: E402
from paper_1811_11842_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", type=int, nargs="+", default=[256, 1024, 4096, 16384])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
BYTES = {"ch": 24.0, "poisson": 16.0}
for n in a.sizes:
    g = torch.Generator(device="cuda").manual_seed(n)
    phi = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    sim = Simulation(n, n, Lambda=1e-5)
    sim.set_fields(phi=phi.contiguous())
    x = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    for op in ("ch", "poisson"):
        sim.reset_stats()
        sim.enable_timing(1)
        for _ in range(a.reps):
            sim.apply_operator(op, x)
        st = sim.stats()
        sim.enable_timing(0)
        kc = st["kernels"]["ch_apply" if op == "ch" else "op_apply"]
        # class timing covers the stencil launch only (not the coefficient kernels)
        ms = kc["ms"] / max(kc["timed"], 1)
        gbs = BYTES[op] * n * n / (ms * 1e-3) / 1e9 if ms > 0 else None
        print(json.dumps({"op": op, "n": n, "ms_per_apply": ms, "GBps": gbs,
                          "bytes_per_cell": BYTES[op]}), flush=True)
    sim.close()
