"""Per-CTA phase timing of one steady-state k_cgs_iter launch (experiments).
Needs a library built with -DCHB_TRACE=1 (scripts/build_variant.sh trace
-DCHB_TRACE=1) selected by CHB_LIB.  Runs an isolated solve, dumps the trace
of the last real sweep and prints phase statistics as one JSON line.
    CHB_LIB=.../libch_b200_trace.so python scripts/trace_sweep.py --solve poisson --config 3
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1811_11842_b200 import Simulation, _lib  # noqa: E402
from workloads import CONFIGS, initial_fields  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--solve", default="poisson")
ap.add_argument("--nb", type=int, default=740)
a = ap.parse_args()
cfg = CONFIGS[a.config]
n, m = cfg["ny"], cfg["nx"]
sim = Simulation(m, n, dt=cfg["dt"])
sim.set_fields(**initial_fields(m, n, seed=0))
import torch  # noqa: E402
g = torch.Generator(device="cuda").manual_seed(3)
b = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
if a.solve == "poisson":
    b -= b.mean()
if a.solve == "mom_v":
    b[0] = 0.0  # the v wall row is not an unknown
x = sim.solve(a.solve, b)
path = "/tmp/chb_trace.bin"
rc = _lib.lib.chb_trace_dump(path.encode(), a.nb)
assert rc == 0, rc
# points: 0 entry, 1 after griddepcontrol.wait, 2 ring ready, 3 row loop end,
# 4 end (after the finalize in the last CTA), 5 reduction entry, 6 after the
# ticket atomic, 7 last CTA: partial sums loaded and summed
raw = np.fromfile(path, dtype=np.uint8)
t = raw[: a.nb * 128].view(np.uint64).reshape(a.nb, 16).astype(np.int64)
smid = raw[a.nb * 128: a.nb * 132].view(np.uint32)
order_raw = raw[a.nb * 132: a.nb * 136].view(np.uint32) if raw.size >= a.nb * 136 else None
gt, ck = t[:, :8], t[:, 8:]
base = gt[:, 0].min()
rel = (gt - base) / 1e3  # us
last = int(np.argmax(gt[:, 4]))
out = {"solve": a.solve, "config": cfg["name"], "nb": a.nb,
       "gt_us": {f"p{i}": [round(float(np.min(rel[:, i])), 3), round(float(np.median(rel[:, i])), 3),
                           round(float(np.max(rel[:, i])), 3)] for i in range(7)},
       "last_cta": last,
       "last_cta_gt_us": [round(float(v), 3) for v in rel[last]],
       "last_cta_cycles_from_p3": [int(v) for v in (ck[last] - ck[last, 3])]}
# per-SM view: row-loop time (p3 - p2) of the CTAs on each SM
loop = rel[:, 3] - rel[:, 2]
per_sm = {}
for b in range(a.nb):
    per_sm.setdefault(int(smid[b]), []).append(float(loop[b]))
sm_mean = np.array([np.mean(v) for v in per_sm.values()])
within = np.mean([np.std(v) for v in per_sm.values()])
out["loop_us"] = [round(float(loop.min()), 2), round(float(np.median(loop)), 2), round(float(loop.max()), 2)]
out["per_sm"] = {"n_sm": len(per_sm), "ctas_per_sm": sorted({len(v) for v in per_sm.values()}),
                 "sm_mean_loop_us": [round(float(sm_mean.min()), 2), round(float(np.median(sm_mean)), 2),
                                     round(float(sm_mean.max()), 2)],
                 "std_across_sm_means": round(float(sm_mean.std()), 2),
                 "mean_std_within_sm": round(float(within), 2),
                 "sm_means_by_smid": {str(k): round(float(np.mean(v)), 2) for k, v in sorted(per_sm.items())}}
if order_raw is not None:
    # row-loop end time and loop duration by dispatch order on the SM
    per = max(1, a.nb // max(1, len(per_sm)))
    order = (order_raw % per).astype(int)
    out["by_order"] = {str(o): {"n": int((order == o).sum()),
                                "loop_us_mean": round(float(loop[order == o].mean()), 2),
                                "loop_end_us_mean": round(float(rel[order == o, 3].mean()), 2),
                                "loop_end_us_max": round(float(rel[order == o, 3].max()), 2)}
                       for o in range(per) if (order == o).any()}
print(json.dumps(out))
