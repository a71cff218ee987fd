"""Per-kernel-class timing of full time steps (CUDA events inside the library).

    CHB_VEC=2 python scripts/kbench.py [--config 3] [--steps 1] [--warmup 1]
Prints one JSON line: per class launches / avg ms / GB/s (algorithmic bytes), iterations.
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
a = ap.parse_args()
cfg = CONFIGS[a.config]
sim = Simulation(cfg["nx"], cfg["ny"], dt=cfg["dt"])
sim.set_fields(**initial_fields(cfg["nx"], cfg["ny"], seed=0))
sim.step(a.warmup)
sim.reset_stats()
sim.enable_timing(a.stride)
sim.step(a.steps)
st = sim.stats()
out = {"variant": os.environ.get("CHB_VEC", "default"), "config": cfg["name"],
       "iters": st["iters_last"], "kernels": {}}
for k, v in st["kernels"].items():
    if v["timed"]:
        out["kernels"][k] = {"launches": v["launches"], "avg_us": 1e3 * v["ms"] / v["timed"],
                             "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9,
                             "total_ms_est": v["ms"] / v["timed"] * v["launches"]}
print(json.dumps(out), flush=True)
sim.close()
