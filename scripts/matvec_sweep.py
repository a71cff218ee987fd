"""BASELINE.json configs[4], second part: isolated CH / Poisson stencil applies
on random fields, 256^2 .. 16384^2 (paper_1811_11842_b200/matvec.py).

    python scripts/matvec_sweep.py [--sizes 256 1024 4096 16384] [--reps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1811_11842_b200.matvec import sweep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", type=int, nargs="+", default=[256, 1024, 4096, 16384])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
for rec in sweep(a.sizes, a.reps):
    print(json.dumps(rec), flush=True)
