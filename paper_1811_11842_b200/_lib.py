"""ctypes binding of include/ch_b200.h (argument marshalling only).

Every step of the hot path runs in libch_b200.so (hand-written sm_100a CUDA);
this module only declares the C structs / prototypes and converts numpy
(host) or torch CUDA (device) arrays to pointers.  There is no CPU fallback:
if the library is missing this module raises at import.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHB_LIB") or os.path.join(HERE, "libch_b200.so")  # override: experiments

CH_OK, CH_ERR_ARG, CH_ERR_CUDA, CH_ERR_NOT_CONVERGED, CH_ERR_BREAKDOWN, CH_ERR_COMM = range(6)
CH_HOST, CH_DEVICE = 0, 1
FIELDS = {"phi": 0, "phi_prev": 1, "c": 2, "u": 3, "v": 4, "p": 5, "u_star": 6, "v_star": 7}
SYSTEMS = ("ch", "nutrient", "u", "v", "p")
OPS = {"ch": 0, "poisson": 1, "mom_u": 2, "mom_v": 3, "nutrient": 4}
SOLVERS = {"bicgstab": 0, "gmres": 1}
KERNEL_CLASSES = ("cg_A", "cg_B", "cg_init", "ch_apply", "vec", "rhs", "gmres", "cg_fused_c",
                  "cg_fused_u", "cg_fused_v", "cg_fused_p", "cg_px", "op_apply")


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("device", C.c_int32), ("virtual_slabs", C.c_int32)]


class Params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("dt", "Gamma1", "Gamma2", "Lambda", "mu", "Kc", "eps",
                                          "A", "Ds", "Re_s", "Re_n", "rho_n", "rho_s", "lid_u",
                                          "rtol", "theta_ch", "theta_adv", "theta_visc")] + \
               [("maxit", C.c_int32), ("ch_solver", C.c_int32), ("gmres_restart", C.c_int32),
                ("refine", C.c_int32), ("startup_be", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("iters_last", C.c_int32 * 5), ("iters_total", C.c_int64 * 5),
                ("resid_last", C.c_double * 5), ("launches", C.c_int64),
                ("kc_launches", C.c_int64 * 16), ("kc_timed", C.c_int64 * 16),
                ("kc_ms", C.c_double * 16), ("kc_bytes", C.c_double * 16)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built -- run __graft_entry__.build() "
                      "(python -m paper_1811_11842_b200.build); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)
_P = C.c_void_p
_D = C.POINTER(C.c_double)
lib.ch_create.restype = _P
lib.ch_create.argtypes = [C.POINTER(Grid), C.POINTER(Params), C.POINTER(C.c_int)]
lib.ch_destroy.restype = None
lib.ch_destroy.argtypes = [_P]
lib.ch_last_error.restype = C.c_char_p
lib.ch_last_error.argtypes = [_P]
lib.ch_abi_version.restype = C.c_int
lib.ch_comm_unique_id.argtypes = [_P, C.c_size_t]
lib.ch_comm_init.argtypes = [_P, _P, C.c_size_t]
lib.ch_local_rows.argtypes = [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
lib.ch_partition.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                             C.POINTER(C.c_int32)]
lib.ch_set_stream.argtypes = [_P, _P]
lib.ch_set_fields.argtypes = [_P, _P, _P, _P, _P, _P, C.c_int]
lib.ch_set_field.argtypes = [_P, C.c_int, _P, C.c_int]
lib.ch_get_fields.argtypes = [_P, _P, _P, _P, _P, _P, C.c_int]
lib.ch_get_field.argtypes = [_P, C.c_int, _P, C.c_int]
lib.ch_step.argtypes = [_P, C.c_int]
lib.ch_apply_operator.argtypes = [_P, C.c_int, _P, _P, C.c_int]
lib.ch_solve.argtypes = [_P, C.c_int, _P, _P, C.c_int]
lib.ch_get_stats.argtypes = [_P, C.POINTER(Stats)]
lib.ch_reset_stats.argtypes = [_P]
lib.ch_enable_timing.argtypes = [_P, C.c_int]
lib.ch_set_time_index.argtypes = [_P, C.c_int64]
lib.ch_get_time_index.argtypes = [_P, C.POINTER(C.c_int64)]
lib.ch_comm_mode.argtypes = [_P]
lib.ch_selftest_xrank.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P]

# every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = ("ch_create", "ch_comm_unique_id", "ch_comm_init", "ch_local_rows", "ch_partition", "ch_set_stream",
           "ch_set_fields", "ch_set_field", "ch_step", "ch_get_fields", "ch_get_field",
           "ch_apply_operator", "ch_solve", "ch_get_stats", "ch_reset_stats", "ch_enable_timing",
           "ch_last_error", "ch_abi_version", "ch_destroy", "ch_set_time_index",
           "ch_get_time_index", "ch_comm_mode", "ch_selftest_xrank")


class CHError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
