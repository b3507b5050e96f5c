"""ctypes wrapper of the CPU oracle (oracle/kkt_oracle.c) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) import
this module, and only as the checker or the CPU timing baseline.  The product path
(paper_2401_13926_b200) never imports it.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libkkt_oracle.so")

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class _System(C.Structure):
    _fields_ = [("n", C.c_int64), ("k_rp", i64p), ("k_ci", i64p), ("k_v", f64p),
                ("k_sym", C.c_int), ("row_perm", i64p), ("col_perm", i64p), ("Lp", i64p),
                ("Li", i64p), ("Up", i64p), ("Ui", i64p), ("Lx", f64p), ("Ux", f64p),
                ("udiag", f64p)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(
                os.path.join(HERE, "kkt_oracle.c")):
            build()
        lib = C.CDLL(LIB)
        lib.oracle_inf_norm.restype = C.c_double
        lib.oracle_fgmres.restype = C.c_int
        lib.oracle_refine_fgmres.restype = C.c_int
        _lib = lib
    return _lib


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(i64p)


def _f(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(f64p)


class OracleFactors:
    """LuFactors arrays (numpy) + the oracle's refactorize / lu_solve."""

    def __init__(self, arrays: dict, general_row_ptr):
        self.a = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
        self.a["Lx"] = self.a["Lx"].astype(np.float64).copy()
        self.a["Ux"] = self.a["Ux"].astype(np.float64).copy()
        self.a["Udiag"] = self.a["Udiag"].astype(np.float64).copy()
        self.g_rp = np.ascontiguousarray(general_row_ptr, dtype=np.int64)
        self.n = self.a["row_perm"].size

    def refactorize(self, general_values) -> np.ndarray:
        lib = load()
        a = self.a
        av, avp = _f(general_values)
        d = np.zeros(4)
        P = lambda k: a[k].ctypes.data_as(i64p if a[k].dtype == np.int64 else f64p)  # noqa: E731
        lib.oracle_refactorize(C.c_int64(self.n), self.g_rp.ctypes.data_as(i64p), avp,
                               C.c_int64(av.size), P("Lp"), P("Li"), P("Lx"), P("Up"),
                               P("Ui"), P("Ux"), P("Udiag"), P("so_ptr"), P("so_data"),
                               P("ap_ptr"), P("a_src"), P("a_tgt"), d.ctypes.data_as(f64p))
        return d

    def lu_solve(self, b) -> np.ndarray:
        lib = load()
        a = self.a
        bb, bp = _f(b)
        x = np.empty(self.n)
        P = lambda k: a[k].ctypes.data_as(i64p if a[k].dtype == np.int64 else f64p)  # noqa: E731
        lib.oracle_lu_solve(C.c_int64(self.n), P("row_perm"), P("col_perm"), P("Lp"), P("Li"),
                            P("Lx"), P("Up"), P("Ui"), P("Ux"), P("Udiag"), bp,
                            x.ctypes.data_as(f64p))
        return x

    def system(self, K_rp, K_ci, K_v, sym_lower=True):
        keep = [_i(K_rp), _i(K_ci), _f(K_v)]
        a = self.a
        P = lambda k: a[k].ctypes.data_as(i64p if a[k].dtype == np.int64 else f64p)  # noqa: E731
        s = _System(self.n, keep[0][1], keep[1][1], keep[2][1], 1 if sym_lower else 0,
                    P("row_perm"), P("col_perm"), P("Lp"), P("Li"), P("Up"), P("Ui"),
                    P("Lx"), P("Ux"), P("Udiag"))
        s._keep = keep
        return s

    def refine_fgmres(self, K_rp, K_ci, K_v, r, x0, delta, m=10, max_outer=10, sym_lower=True):
        lib = load()
        S = self.system(K_rp, K_ci, K_v, sym_lower)
        rr, rp = _f(r)
        xx, xp = _f(x0)
        x = np.empty(self.n)
        out = np.zeros(6)
        rc = lib.oracle_refine_fgmres(C.byref(S), rp, xp, m, max_outer, C.c_double(delta),
                                      x.ctypes.data_as(f64p), out.ctypes.data_as(f64p))
        if rc:
            raise FloatingPointError("oracle fgmres: non-finite operator output")
        return x, dict(triggered=bool(out[0]), iterations=int(out[1]), converged=bool(out[2]),
                       nsr_before=out[3], nsr_after=out[4], rr_final=out[5])


def spmv(K_rp, K_ci, K_v, x, sym_lower=True) -> np.ndarray:
    lib = load()
    rp, rpp = _i(K_rp)
    ci, cip = _i(K_ci)
    v, vp = _f(K_v)
    xx, xp = _f(x)
    y = np.empty(rp.size - 1)
    lib.oracle_spmv(C.c_int64(rp.size - 1), rpp, cip, vp, 1 if sym_lower else 0, xp,
                    y.ctypes.data_as(f64p))
    return y


def inf_norm(K_rp, K_ci, K_v, sym_lower=True) -> float:
    lib = load()
    rp, rpp = _i(K_rp)
    ci, cip = _i(K_ci)
    v, vp = _f(K_v)
    return lib.oracle_inf_norm(C.c_int64(rp.size - 1), rpp, cip, vp, 1 if sym_lower else 0)
