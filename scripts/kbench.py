"""Per-kernel-class timing (CUDA events inside the library) of full time steps,
or of isolated solves of one operator.

    CHB_DEFER=8 python scripts/kbench.py [--config 3] [--steps 1] [--warmup 1]
    python scripts/kbench.py --solve poisson|mom_u|mom_v [--config 3]
Prints one JSON line: per class launches / avg us / GB/s (algorithmic bytes), iterations.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1811_11842_b200 import Simulation  # noqa: E402
from workloads import CONFIGS, initial_fields  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--stride", type=int, default=4)
ap.add_argument("--solve", default=None)
ap.add_argument("--nx", type=int, default=0, help="override the config's grid (e.g. one rank's slab)")
ap.add_argument("--ny", type=int, default=0)
a = ap.parse_args()
cfg = dict(CONFIGS[a.config])
if a.nx and a.ny:
    cfg.update(nx=a.nx, ny=a.ny, name=f"{a.nx}x{a.ny}")
sim = Simulation(cfg["nx"], cfg["ny"], dt=cfg["dt"])
sim.set_fields(**initial_fields(cfg["nx"], cfg["ny"], seed=0))
if a.solve:
    import torch
    n, m = cfg["ny"], cfg["nx"]
    g = torch.Generator(device="cuda").manual_seed(3)
    b = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
    if a.solve == "poisson":
        b -= b.mean()
    if a.solve == "mom_v":
        b[0] = 0.0
    sim.solve(a.solve, b)          # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.solve(a.solve, b)          # untimed per kernel: the solve's own wall time
    e1.record()
    torch.cuda.synchronize()
    solve_ms = e0.elapsed_time(e1)
    sim.reset_stats()
    sim.enable_timing(a.stride)
    sim.solve(a.solve, b)
else:
    sim.step(a.warmup)
    sim.reset_stats()
    sim.enable_timing(a.stride)
    sim.step(a.steps)
st = sim.stats()
out = {"lib": os.environ.get("CHB_LIB", "default"), "defer": os.environ.get("CHB_DEFER", "64"),
       "solve": a.solve, "config": cfg["name"], "iters": st["iters_last"], "kernels": {}}
if a.solve:
    out["solve_ms"] = solve_ms
for k, v in st["kernels"].items():
    if v["timed"]:
        out["kernels"][k] = {"launches": v["launches"], "avg_us": 1e3 * v["ms"] / v["timed"],
                             "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9,
                             "total_ms_est": v["ms"] / v["timed"] * v["launches"]}
print(json.dumps(out), flush=True)
sim.close()
