"""Write tests/golden/oracle_<n>_<steps>.npz by running ONLY the CPU oracle
(oracle/) on the seeded BASELINE.json configs[1] initial condition.

    python scripts/gen_golden.py 256 100
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Params, initial_state, step  # noqa: E402
from workloads import initial_fields  # noqa: E402


def main(n=256, steps=100, seed=0, rtol=1e-10):
    st = initial_state(initial_fields(n, n, seed=seed))
    prm = Params(rtol=rtol)
    t0 = time.time()
    iters = []
    for k in range(steps):
        st, info = step(st, prm)
        iters.append([info.iters[s] for s in ("ch", "nutrient", "u", "v", "p")])
        if k % 10 == 0:
            print(k, info.iters, f"{time.time() - t0:.0f}s", flush=True)
    tag = "" if rtol == 1e-10 else f"_rtol{rtol:.0e}"
    out = os.path.join(ROOT, "tests", "golden", f"oracle_{n}_{steps}{tag}.npz")
    np.savez_compressed(out, phi=st.phi, c=st.c, u=st.u, v=st.v, p=st.p,
                        phi_prev=st.phi_prev, iters=np.array(iters), seed=seed, rtol=rtol,
                        note="oracle/ fp64, BASELINE.json configs[1] (256^2, 100 steps, dt=1e-4)")
    print("wrote", out)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 256, int(a[1]) if len(a) > 1 else 100, 0,
         float(a[2]) if len(a) > 2 else 1e-10)
