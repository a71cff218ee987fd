"""Multi-process plumbing for the slab decomposition in y (one process per
GPU, torch.distributed for the host-side collectives; the data path -- halo
rows and Krylov partial sums -- runs inside libch_b200.so over NCCL).

Everything here is backend-agnostic host logic (gloo on CPU in the tests,
NCCL on the GPU box): which rows a rank owns (the library's own
ch_partition), the NCCL clique id broadcast, gathering slabs into a global
field and the max-over-ranks timing reduction bench.py reports.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def partition(ny: int, nranks: int, rank: int, virtual_slabs: int = 1) -> tuple[int, int]:
    """(row0, nrows) of `rank` -- the decomposition ch_create applies."""
    r0, nr = C.c_int32(), C.c_int32()
    rc = _lib.lib.ch_partition(ny, nranks, rank, virtual_slabs, C.byref(r0), C.byref(nr))
    if rc != _lib.CH_OK:
        raise ValueError(f"invalid decomposition ny={ny} nranks={nranks} slabs={virtual_slabs}")
    return r0.value, nr.value


def share_unique_id(dist, rank: int) -> bytes:
    """Rank 0 creates the NCCL clique id (ch_comm_unique_id); everyone gets it."""
    from . import unique_id
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(dist, value: float, device=None) -> float:
    """Max of a per-rank scalar (device-timed ms) -- the bench's job time."""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(dist, local: np.ndarray, ny: int, world: int) -> np.ndarray | None:
    """Assemble the (ny, nx) global field from every rank's (nrows, nx) slab
    (rank order = row order).  Returns the field on every rank."""
    import torch
    nx = local.shape[1]
    parts = [partition(ny, world, r) for r in range(world)]
    hmax = max(nr for _, nr in parts)
    buf = torch.zeros((hmax, nx), dtype=torch.float64)
    buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local))
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return np.concatenate([out[r][: parts[r][1]].numpy() for r in range(world)], axis=0)
