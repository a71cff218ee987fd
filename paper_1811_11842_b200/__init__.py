"""B200-native hot path of arxiv 1811.11842 (2D biofilm: modified Cahn-Hilliard
+ Chorin projection) behind the C ABI of include/ch_b200.h.

    from paper_1811_11842_b200 import Simulation
    sim = Simulation(256, 256)                 # PAPER.md §5 parameters, dt = 1e-4
    sim.set_fields(phi=phi0, c=c0, u=u0, v=v0, p=p0)   # numpy (host) or torch.cuda (device)
    sim.step(100)
    out = sim.get_fields()                     # dict of numpy arrays

The Python layer only marshals arguments; all arithmetic runs in
libch_b200.so.  PyTorch (optional) supplies device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields as dc_fields

import numpy as np

from . import _lib
from ._lib import CHError, lib

__all__ = ["Simulation", "SimParams", "CHError", "unique_id"]


@dataclass
class SimParams:
    """ch_params with PAPER.md §5 defaults (lines 271-274), R8-R10, R13;
    theta_* = implicit weights (R5, R7, R12), startup_be = backward-Euler
    start-up steps (R23); refine = CG restarts until the true residual meets
    rtol (R21, 0 = off)."""
    dt: float = 1e-4
    Gamma1: float = 33.467
    Gamma2: float = 1.25e6
    Lambda: float = 1e-10
    mu: float = 0.14
    Kc: float = 0.15
    eps: float = 1.0
    A: float = 100.0
    Ds: float = 2.3
    Re_s: float = 9.98e-4
    Re_n: float = 2.33e-9
    rho_n: float = 1.0
    rho_s: float = 1.0
    lid_u: float = 1.0
    rtol: float = 1e-10
    theta_ch: float = 0.5
    theta_adv: float = 0.5
    theta_visc: float = 1.0
    maxit: int = 200000
    ch_solver: str = "bicgstab"
    gmres_restart: int = 30
    refine: int = 0
    startup_be: int = 2

    def to_c(self) -> _lib.Params:
        p = _lib.Params()
        for f in dc_fields(self):
            v = getattr(self, f.name)
            if f.name == "ch_solver":
                v = _lib.SOLVERS[v]
            setattr(p, f.name, v)
        return p


def unique_id() -> bytes:
    """128-byte NCCL unique id for ch_comm_init (rank 0 creates, caller broadcasts)."""
    buf = C.create_string_buffer(128)
    rc = lib.ch_comm_unique_id(buf, 128)
    if rc != 0:
        raise CHError(rc, "ncclGetUniqueId failed")
    return buf.raw


def _ptr(a, shape):
    """(pointer, where) of a host numpy or device torch array with the expected shape."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous or a.shape != shape:
            raise ValueError(f"expected C-contiguous float64 {shape}, got {a.dtype} {a.shape}")
        return a.ctypes.data, _lib.CH_HOST
    if getattr(a, "is_cuda", False):
        import torch
        if a.dtype != torch.float64 or not a.is_contiguous() or tuple(a.shape) != shape:
            raise ValueError(f"expected contiguous float64 cuda {shape}, got {a.dtype} {tuple(a.shape)}")
        return a.data_ptr(), _lib.CH_DEVICE
    raise TypeError("arrays must be numpy (host) or torch CUDA tensors (device)")


class Simulation:
    def __init__(self, nx: int, ny: int, params: SimParams | None = None, *, rank: int = 0,
                 nranks: int = 1, device: int = 0, virtual_slabs: int = 1, **overrides):
        self.params = params or SimParams()
        for k, v in overrides.items():
            setattr(self.params, k, v)
        g = _lib.Grid(nx, ny, rank, nranks, device, virtual_slabs)
        st = C.c_int(0)
        self._h = lib.ch_create(C.byref(g), C.byref(self.params.to_c()), C.byref(st))
        if not self._h:
            raise CHError(st.value, "ch_create failed (see stderr)")
        self.nx, self.ny = nx, ny
        r0, nr = C.c_int32(), C.c_int32()
        lib.ch_local_rows(self._h, C.byref(r0), C.byref(nr))
        self.row0, self.nrows = r0.value, nr.value

    # -- helpers
    def _check(self, rc):
        if rc != _lib.CH_OK:
            raise CHError(rc, lib.ch_last_error(self._h).decode())

    @property
    def shape(self):
        return (self.nrows, self.nx)

    def comm_init(self, uid: bytes):
        self._check(lib.ch_comm_init(self._h, uid, len(uid)))

    @property
    def comm_mode(self) -> str:
        """"single" (one process), "nccl" (NCCL group per CG iteration) or
        "p2p" (peer-memory CG iterations, ch_comm_mode)."""
        if not self._h:
            raise CHError(_lib.CH_ERR_ARG, "simulation is closed")
        return {0: "single", 1: "nccl", 2: "p2p"}[lib.ch_comm_mode(self._h)]

    def set_stream(self, stream):
        """stream: torch.cuda.Stream, raw cudaStream_t int, or None (legacy default)."""
        ptr = getattr(stream, "cuda_stream", stream)
        self._check(lib.ch_set_stream(self._h, ptr))

    # -- state
    def set_fields(self, phi=None, c=None, u=None, v=None, p=None):
        ptrs, where = [], None
        for a in (phi, c, u, v, p):
            if a is None:
                ptrs.append(None)
                continue
            ptr, w = _ptr(a, self.shape)
            if where is not None and w != where:
                raise ValueError("mix of host and device arrays")
            where = w
            ptrs.append(ptr)
        self._check(lib.ch_set_fields(self._h, *ptrs, _lib.CH_HOST if where is None else where))

    def set_field(self, name: str, a):
        ptr, w = _ptr(a, self.shape)
        self._check(lib.ch_set_field(self._h, _lib.FIELDS[name], ptr, w))

    def get_field(self, name: str, out=None):
        if out is None:
            out = np.empty(self.shape)
        ptr, w = _ptr(out, self.shape)
        self._check(lib.ch_get_field(self._h, _lib.FIELDS[name], ptr, w))
        return out

    def get_fields(self, names=("phi", "c", "u", "v", "p"), device: bool = False) -> dict:
        out = {}
        for n in names:
            if device:
                import torch
                buf = torch.empty(self.shape, dtype=torch.float64, device="cuda")
            else:
                buf = np.empty(self.shape)
            out[n] = self.get_field(n, buf)
        return out

    @property
    def time_index(self) -> int:
        n = C.c_int64()
        self._check(lib.ch_get_time_index(self._h, C.byref(n)))
        return n.value

    @time_index.setter
    def time_index(self, n: int):
        self._check(lib.ch_set_time_index(self._h, int(n)))

    def step(self, n: int = 1):
        self._check(lib.ch_step(self._h, n))

    def apply_operator(self, op: str, x):
        import copy as _copy
        if isinstance(x, np.ndarray):
            y = np.empty_like(x)
        else:
            y = _copy.copy(x).new_empty(x.shape)
        px, wx = _ptr(x, self.shape)
        py, _ = _ptr(y, self.shape)
        self._check(lib.ch_apply_operator(self._h, _lib.OPS[op], px, py, wx))
        return y

    def solve(self, op: str, b, x0=None):
        """Solve Op x = b (coefficients from the current state) with the step's
        Krylov method for that operator; returns x (same kind of array as b)."""
        import copy as _copy
        if x0 is None:
            x = np.zeros_like(b) if isinstance(b, np.ndarray) else _copy.copy(b).new_zeros(b.shape)
        else:
            x = x0.copy() if isinstance(x0, np.ndarray) else x0.clone()
        pb, wb = _ptr(b, self.shape)
        px, wx = _ptr(x, self.shape)
        if wb != wx:
            raise ValueError("b and x0 must both be host or both be device arrays")
        self._check(lib.ch_solve(self._h, _lib.OPS[op], pb, px, wb))
        return x

    # -- stats / timing
    def enable_timing(self, stride: int = 1):
        self._check(lib.ch_enable_timing(self._h, stride))

    def reset_stats(self):
        self._check(lib.ch_reset_stats(self._h))

    def stats(self) -> dict:
        s = _lib.Stats()
        self._check(lib.ch_get_stats(self._h, C.byref(s)))
        kc = {}
        for i, name in enumerate(_lib.KERNEL_CLASSES):
            kc[name] = dict(launches=s.kc_launches[i], timed=s.kc_timed[i], ms=s.kc_ms[i],
                            bytes=s.kc_bytes[i])
        return dict(steps=s.steps, launches=s.launches,
                    iters_last=dict(zip(_lib.SYSTEMS, list(s.iters_last))),
                    iters_total=dict(zip(_lib.SYSTEMS, list(s.iters_total))),
                    resid_last=dict(zip(_lib.SYSTEMS, list(s.resid_last))),
                    kernels=kc)

    def close(self):
        if getattr(self, "_h", None):
            lib.ch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
