"""The peer-memory combine of the multi-slab CG sweep (common.cuh
xrank_combine) on one GPU: R groups of CTAs play R ranks inside
one cooperative launch (ch_selftest_xrank), each with its own totals area,
flags and peer table, over many iterations with randomised arrival order.
Every rank must compute the slab-ordered sums bit for bit, and a rank that
never arrives must turn into a reported timeout on every other rank, not a
hang.  The product sweep runs the same device function (across processes on
NVLink peer mappings; within one process with R = 1, exercised by every
virtual-slab test)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nranks,nloc", [(1, 1), (1, 4), (2, 1), (3, 2), (4, 2), (8, 1), (8, 8)])
def test_xrank_combine_is_exact_and_identical_on_every_rank(nranks, nloc):
    from paper_1811_11842_b200._lib import lib
    last = (C.c_double * (nranks * 8))()
    bad = lib.ch_selftest_xrank(0, nranks, nloc, 40, 0, last)
    assert bad == 0, bad
    for r in range(1, nranks):
        assert [last[r * 8 + k] for k in range(3)] == [last[k] for k in range(3)]


def test_xrank_absent_rank_times_out_without_hanging():
    from paper_1811_11842_b200._lib import lib
    # epochs 1-2 normal, epoch 2 with the last rank absent (others report a
    # timeout after ~2 s), epoch 3 normal again after the reset
    assert lib.ch_selftest_xrank(0, 3, 2, 3, 2, None) == 0


def test_comm_mode_single_process():
    from paper_1811_11842_b200 import Simulation
    sim = Simulation(16, 16, virtual_slabs=2)
    assert sim.comm_mode == "single"
    sim.close()
