"""Run N time steps at a config size (for ncu captures / launch lists).

    python scripts/prof_step.py [--config 3] [--steps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1811_11842_b200 import Simulation  # noqa: E402
from workloads import CONFIGS, initial_fields  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
cfg = CONFIGS[a.config]
sim = Simulation(cfg["nx"], cfg["ny"], dt=cfg["dt"])
sim.set_fields(**initial_fields(cfg["nx"], cfg["ny"], seed=0))
sim.step(a.steps)
print(sim.stats()["iters_last"])
sim.close()
