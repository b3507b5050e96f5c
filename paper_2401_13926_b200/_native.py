"""ctypes binding of libkktb200.so (the C ABI declared in include/kktb200.h).

The library is built in-tree (``paper_2401_13926_b200/libkktb200.so``).  There is no
fallback: if it is missing or stale-incompatible, importing the solver raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkktb200.so")
ABI_VERSION = 4

KKT_OK = 0
KKT_ERR_SINGULAR = 1
KKT_ERR_PATTERN_MISMATCH = 2
KKT_ERR_BAD_SHAPE = 3
KKT_ERR_NONFINITE = 4
KKT_ERR_CUDA = 5
KKT_ERR_OOM = 6
KKT_ERR_BAD_ARG = 7
KKT_ERR_CALLBACK = 8
FG_STATS_AFTER = 1
FG_HOST_LOOP = 2
FG_MGS = 4
FG_NO_HANDOFF = 8
OP_HANDLE, OP_IDENTITY, OP_MATRIX, OP_CALLBACK = 0, 1, 2, 3
LAYOUT_GENERAL = 0
LAYOUT_SYMMETRIC_LOWER = 1

i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class DeviceOpts(C.Structure):
    _fields_ = [("device", C.c_int), ("batch", C.c_int), ("restart_m", C.c_int),
                ("reserved", C.c_int), ("flags", C.c_int)]


class KrylovCfg(C.Structure):
    _fields_ = [("m", C.c_int), ("max_outer", C.c_int), ("tol", C.c_double),
                ("delta_tol", C.c_double), ("delta_sys", C.POINTER(C.c_double)),
                ("flags", C.c_int)]


class KrylovReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int),
                ("precond_applications", C.c_int), ("restarts", C.c_int),
                ("beta0", C.c_double), ("est_final", C.c_double),
                ("true_final", C.c_double), ("triggered", C.c_int), ("nonfinite", C.c_int),
                ("stats_before", C.c_double * 6), ("stats_after", C.c_double * 6),
                ("handed_off", C.c_int), ("reserved_", C.c_int)]


APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


class LinOp(C.Structure):
    _fields_ = [("kind", C.c_int), ("matrix", C.c_void_p), ("apply", APPLY_FN),
                ("user", C.c_void_p)]


# (name, restype, argtypes) — every symbol include/kktb200.h declares.
SIGNATURES = [
    ("kkt_last_error", C.c_char_p, []),
    ("kkt_abi_version", C.c_int, []),
    ("kkt_analyze", C.c_int, [i64, i64p, i64p, f64p, C.c_double, C.POINTER(vp)]),
    ("kkt_min_degree_order", C.c_int, [i64, i64p, i64p, i64p]),
    ("kkt_symbolic_free", None, [vp]),
    ("kkt_symbolic_sizes", C.c_int, [vp, i64p]),
    ("kkt_symbolic_export", C.c_int, [vp] + [i64p, i64p, i64p, i64p, f64p, i64p, i64p, f64p,
                                           f64p, i64p, i64p, i64p, i64p, i64p]),
    ("kkt_symbolic_diag", C.c_int, [vp, f64p]),
    ("kkt_symbolic_stats", C.c_int, [vp, i64p]),
    ("kkt_dev_create", C.c_int, [vp, i64p, i64p, i64, i64p, C.POINTER(DeviceOpts), C.POINTER(vp)]),
    ("kkt_dev_destroy", None, [vp]),
    ("kkt_plan_check", C.c_int, [vp, i64p, i64p, i64, i64p, i64p]),
    ("kkt_dev_stream", vp, [vp]),
    ("kkt_dev_refactor", C.c_int, [vp, vp, C.c_int, C.c_int, f64p]),
    ("kkt_dev_set_operator_values", C.c_int, [vp, vp, C.c_int, C.c_int]),
    ("kkt_dev_solve", C.c_int, [vp, vp, vp]),
    ("kkt_dev_spmv", C.c_int, [vp, vp, vp]),
    ("kkt_dev_residual_norms", C.c_int, [vp, vp, vp, f64p]),
    ("kkt_dev_residual", C.c_int, [vp, vp, vp, vp, f64p]),
    ("kkt_dev_axpy", C.c_int, [vp, vp, vp]),
    ("kkt_assemble_values", C.c_int, [i64, i64, i64, i64, C.c_int, vp, vp, vp, vp, vp, vp, vp]),
    ("kkt_assemble_rhs", C.c_int, [i64, i64, C.c_int, vp, vp, vp, vp, vp, vp, vp]),
    ("kkt_recover_dz", C.c_int, [i64, C.c_int, i64, vp, vp, vp, vp, vp, vp]),
    ("kkt_mm_info", C.c_int, [C.c_char_p, i64p]),
    ("kkt_mm_read_coo", C.c_int, [C.c_char_p, i64, i64p, i64p, f64p]),
    ("kkt_mm_read_array", C.c_int, [C.c_char_p, i64, f64p]),
    ("kkt_dev_fgmres", C.c_int, [vp, vp, vp, vp, C.POINTER(KrylovCfg), C.POINTER(KrylovReport),
                                 f64p, C.c_int]),
    ("kkt_dev_fgmres_ops", C.c_int, [vp, C.POINTER(LinOp), C.POINTER(LinOp), vp, vp, vp,
                                     C.POINTER(KrylovCfg), C.POINTER(KrylovReport), f64p, C.c_int,
                                     f64p, C.c_int]),
    ("kkt_dev_refine_fgmres", C.c_int, [vp, vp, vp, vp, C.POINTER(KrylovCfg),
                                        C.POINTER(KrylovReport)]),
    ("kkt_dev_step", C.c_int, [vp, vp, C.c_int, vp, vp, C.c_int, C.POINTER(KrylovCfg),
                               C.POINTER(KrylovReport), f64p]),
    ("kkt_dev_step_solve", C.c_int, [vp, vp, vp, C.c_int, C.POINTER(KrylovCfg), C.POINTER(KrylovReport)]),
    ("kkt_dev_download_factors", C.c_int, [vp, f64p, f64p, f64p]),
    ("kkt_dev_upload_factors", C.c_int, [vp, f64p, f64p, f64p]),
    ("kkt_op_create", C.c_int, [i64, i64p, i64p, C.c_int, C.c_int, C.POINTER(vp)]),
    ("kkt_op_destroy", None, [vp]),
    ("kkt_op_stream", vp, [vp]),
    ("kkt_op_set_values", C.c_int, [vp, vp, C.c_int]),
    ("kkt_op_spmv", C.c_int, [vp, vp, vp]),
    ("kkt_op_residual_norms", C.c_int, [vp, vp, vp, f64p]),
    ("kkt_dev_info", C.c_int, [vp, i64p]),
    ("kkt_dev_trace", C.c_int, [vp, vp, vp]),
    ("kkt_dev_trace_steps", C.c_int, [vp, vp]),
    ("kkt_dev_launch_count", i64, [vp]),
    ("kkt_probe_hop_ns", C.c_int, [C.c_int, C.c_int, f64p]),
    ("kkt_dev_solve_native", C.c_int, [vp, vp, vp]),
    ("kkt_dev_spmv_native", C.c_int, [vp, vp, vp]),
]

_lib = None


def load():
    """Load (and type) the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2401_13926_b200.build` "
            "(there is no CPU fallback for the solver path)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.kkt_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI version {lib.kkt_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().kkt_last_error()
    return msg.decode() if msg else ""


def ptr_i64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(i64p)


def ptr_f64(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(f64p)


def check(rc: int, what: str = "") -> None:
    """Map a status code to the reference's exception classes."""
    if rc == KKT_OK:
        return
    msg = last_error() or what
    from .direct_lu import PatternMismatchError, SingularMatrixError
    from .krylov import OperatorOutputError
    if rc == KKT_ERR_SINGULAR:
        raise SingularMatrixError(msg)
    if rc == KKT_ERR_PATTERN_MISMATCH:
        raise PatternMismatchError(msg)
    if rc in (KKT_ERR_BAD_SHAPE, KKT_ERR_BAD_ARG):
        raise ValueError(msg)
    if rc == KKT_ERR_NONFINITE:
        raise OperatorOutputError(msg)
    if rc == KKT_ERR_CALLBACK:
        raise RuntimeError(f"operator callback failed: {msg}")
    if rc == KKT_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(f"kktb200 CUDA error: {msg}")
