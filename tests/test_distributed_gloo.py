"""World-size-2 tests of the multi-process (slab-in-y) host path on CPU with
the gloo backend: the decomposition the library applies, the per-rank input
slabs, slab gathering and the max-over-ranks timing reduction (-m "not gpu").
The device data path (halo rows, Krylov partial sums over NCCL) is covered on
one GPU by the virtual-slab parity tests (tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world, dist)))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


def _slabs_tile_global(rank, world, dist):
    from paper_1811_11842_b200.distributed import gather_rows, partition
    from workloads import initial_fields
    nx, ny = 48, 37
    r0, nr = partition(ny, world, rank)
    f = initial_fields(nx, ny, seed=7, rows=(r0, r0 + nr))
    glob = gather_rows(dist, f["phi"], ny, world)
    ref = initial_fields(nx, ny, seed=7)["phi"]
    return bool(np.array_equal(glob, ref)), (r0, nr)


def test_slab_inputs_gather_to_global_field():
    res = _run(_slabs_tile_global)
    assert all(r[0] is True for r in res.values()), res
    (r00, n0), (r01, n1) = res[0][1], res[1][1]
    assert r00 == 0 and r01 == n0 and n0 + n1 == 37 and abs(n0 - n1) <= 1


def _timing_max(rank, world, dist):
    from paper_1811_11842_b200.distributed import max_over_ranks
    return max_over_ranks(dist, 10.0 + 5.0 * rank)


def test_job_time_is_max_over_ranks():
    res = _run(_timing_max)
    assert res == {0: 15.0, 1: 15.0}


def _partition_all(rank, world, dist):
    from paper_1811_11842_b200.distributed import partition
    out = {}
    for ny in (4, 5, 37, 4096):
        for slabs in (1, 2):
            try:
                out[(ny, slabs)] = partition(ny, world, rank, slabs)
            except ValueError:
                out[(ny, slabs)] = None
    return out


def test_partition_consistent_across_ranks():
    res = _run(_partition_all)
    for key in res[0]:
        a, b = res[0][key], res[1][key]
        ny, slabs = key
        if ny < 2 * 2 * slabs:
            assert a is None and b is None
            continue
        assert a[0] == 0 and a[0] + a[1] == b[0] and b[0] + b[1] == ny, (key, a, b)
        assert a[1] >= 2 * slabs and b[1] >= 2 * slabs
