"""Write tests/golden/oracle_<n>_<steps>[_rtolX][_subK].npz by running ONLY the
CPU oracle (oracle/) on the seeded BASELINE.json initial condition.

    python scripts/gen_golden.py 256 100                 # configs[1], full fields
    python scripts/gen_golden.py 256 100 1e-12           # same at rtol 1e-12
    python scripts/gen_golden.py 512 25 1e-10 2          # every 2nd point per direction
    python scripts/gen_golden.py 1024 1 1e-12 4          # configs[2] size, one step

With sub = K > 1 the file keeps the fields at rows/columns 0, K, 2K, ... plus
each full field's L2 norm (the GPU test compares the same subsample).
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Params, initial_state, step  # noqa: E402
from workloads import initial_fields  # noqa: E402


def main(n=256, steps=100, seed=0, rtol=1e-10, sub=1):
    st = initial_state(initial_fields(n, n, seed=seed))
    prm = Params(rtol=rtol)
    t0 = time.time()
    iters = []
    for k in range(steps):
        st, info = step(st, prm)
        iters.append([info.iters[s] for s in ("ch", "nutrient", "u", "v", "p")])
        print(k, info.iters, f"{time.time() - t0:.0f}s", flush=True)
    tag = "" if rtol == 1e-10 else f"_rtol{rtol:.0e}"
    tag += "" if sub == 1 else f"_sub{sub}"
    out = os.path.join(ROOT, "tests", "golden", f"oracle_{n}_{steps}{tag}.npz")
    fields = {k: getattr(st, k) for k in ("phi", "c", "u", "v", "p", "phi_prev")}
    norms = {f"norm_{k}": np.linalg.norm(v) for k, v in fields.items()}
    np.savez_compressed(out, **{k: v[::sub, ::sub] for k, v in fields.items()}, **norms,
                        iters=np.array(iters), seed=seed, rtol=rtol, sub=sub, steps=steps,
                        note=f"oracle/ fp64, BASELINE.json initial condition ({n}^2, {steps} "
                             f"steps, dt={prm.dt}), every {sub}-th point")
    print("wrote", out, f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 256, int(a[1]) if len(a) > 1 else 100, 0,
         float(a[2]) if len(a) > 2 else 1e-10, int(a[3]) if len(a) > 3 else 1)
