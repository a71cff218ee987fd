"""CPU ORACLE -- test infrastructure only.

A plain, slow, single-threaded fp64 implementation (numpy + scipy.sparse
assembled matrices + textbook Krylov) of one semi-implicit time step of the
paper's 2D biofilm model (arxiv 1811.11842, §2-§4), written from the
paper's equations in its order and notation.  It exists to prove the CUDA
path right; it is NOT part of the product:

  * only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import it;
  * it shares no code with ``paper_1811_11842_b200/`` (no kernels, headers,
    helpers, constants or pre/post-processing); the only shared module is
    ``workloads/`` (seeded input generators, no method arithmetic).

Every function cites the PAPER.md passage it follows ("PAPER.md:<line>",
section / equation).  The readings taken where the paper is silent or garbled
are listed in DESIGN.md §3 ("R1".."R20") and cited here by tag.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie it to things other than
itself: exact discrete eigenpairs, closed-form one-step amplification factors,
manufactured-solution convergence order, telescoping mass conservation, free
energy decay, discrete divergence-free projection, dense direct solves,
brute-force loop stencils on tiny grids, and the paper's printed numbers
(Listing 3's 5-point values, §5's dimensionless parameters from Table 1).
No oracle function is "parity unpinned".
"""
from threadpoolctl import threadpool_limits as _tpl

# The oracle is single-threaded by design; OpenBLAS' threaded level-1 kernels
# are also pathologically slow on short vectors in this image (7 ms per dot).
_tpl(1, user_api="blas")

from .params import Params, nondimensionalise  # noqa: F401
from .step import State, step, run, initial_state  # noqa: F401
