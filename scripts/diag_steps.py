#!/usr/bin/env python
"""Per-step field diagnostics of the GPU time step (one JSON line per step).

    python scripts/diag_steps.py --n 4096 --steps 30 [--refine 2] [--set key=val ...]

For each step: Krylov iterations per system, min/max of phi, c, |u|, |v|, the
minimum of the nutrient diagonal (1-phi^{n+1})/dt + A/2 phi^{1/2}, the advective
CFL max(|u|/hx, |v|/hy) dt, and the discrete divergence max.  Used to locate
where a long trajectory leaves the range the discretisation is valid in.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--refine", type=int, default=2)
    ap.add_argument("--set", nargs="*", default=[])
    args = ap.parse_args()
    import torch
    from paper_1811_11842_b200 import CHError, SimParams, Simulation
    from workloads import initial_fields
    n = args.n
    sp = SimParams(refine=args.refine)
    for kv in args.set:
        k, v = kv.split("=")
        setattr(sp, k, type(getattr(sp, k))(v))
    sim = Simulation(n, n, sp)
    sim.set_stream(torch.cuda.current_stream())
    sim.set_fields(**initial_fields(n, n, seed=0))
    prev = sim.get_fields(("phi",), device=True)["phi"]
    for s in range(args.steps):
        t0 = time.time()
        err = None
        try:
            sim.step(1)
        except CHError as e:
            err = str(e)
        torch.cuda.synchronize()
        dt_s = time.time() - t0
        f = sim.get_fields(("phi", "c", "u", "v", "p"), device=True)
        ph, c, u, v = f["phi"], f["c"], f["u"], f["v"]
        half = 0.5 * (ph + prev)
        ac = (1 - ph) / sp.dt + 0.5 * sp.A * half
        ux = u.abs().max().item()
        vx = v.abs().max().item()
        rec = dict(step=s + 1, sec=round(dt_s, 3), err=err,
                   iters=sim.stats()["iters_last"],
                   resid=sim.stats()["resid_last"],
                   phi=[ph.min().item(), ph.max().item()],
                   phi_nan=int(torch.isnan(ph).sum().item()),
                   c=[c.min().item(), c.max().item()],
                   umax=ux, vmax=vx, cfl=max(ux, vx) * n * sp.dt,
                   ac_min=ac.min().item(), mass=ph.mean().item())
        print(json.dumps(rec), flush=True)
        prev = ph
        if err:
            break
    sim.close()


if __name__ == "__main__":
    main()
