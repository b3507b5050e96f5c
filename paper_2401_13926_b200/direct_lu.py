"""Drop-in for ``kktsolve.direct_lu``: analyze on the host, refactor/solve on the B200.

* :func:`factorize`   -> ``kkt_analyze`` (C++, bit-exact with direct_lu.py:116-294)
* :func:`refactorize` -> ``kkt_dev_refactor`` (sm_100a, bitwise with direct_lu.py:297-356)
* :func:`lu_solve`    -> ``kkt_dev_solve`` (sm_100a, bitwise with direct_lu.py:359-379)

``LuFactors`` keeps the reference's field names (``_Lp``, ``_Li``, ``_Lx``, ... ,
``triangular_solve_count``, ``from_refactorization``) so the reference's tests and harness
read it unchanged.  Factor values live on the device after a refactorization; the
``_Lx``/``_Ux``/``_Udiag`` attributes download them lazily.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .sparse import (GENERAL, SYMMETRIC_LOWER, CsMatrix, Permutation, Triplets,
                     expand_pattern, from_triplets)

PATCH_RELATIVE_FLOOR = 1e-12  # direct_lu.py:32


class SingularMatrixError(RuntimeError):
    """No admissible pivot during a first factorization (direct_lu.py:35)."""


class PatternMismatchError(ValueError):
    """refactorize() received a different sparsity pattern (direct_lu.py:39)."""


@dataclass
class LuDiagnostics:
    max_abs_pivot: float
    min_abs_pivot: float
    zero_pivots_patched: int
    growth_estimate: float


class _Symbolic:
    """Owner of the host analysis handle (kkt_symbolic*)."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            try:
                nat.load().kkt_symbolic_free(self.ptr)
            except Exception:
                pass
            self.ptr = None


class LuFactors:
    """LU factors + frozen replay schedule (direct_lu.py:51-107)."""

    def __init__(self):
        self.n = 0
        self.pivot_tol = 0.0
        self.row_perm: Permutation | None = None
        self.col_perm: Permutation | None = None
        self.from_refactorization = False
        self.triangular_solve_count = 0
        self._Lp = self._Li = None
        self._Up = self._Ui = None
        self._so_ptr = self._so_data = None
        self._ap_ptr = self._a_src = self._a_tgt = None
        self._pattern_ref: CsMatrix | None = None
        self._host_vals = None          # (Lx, Ux, Udiag) numpy, or None when device is newer
        self._sym: _Symbolic | None = None
        self._dev = None                # DeviceSystem, created on first device use
        self._L_cache = None
        self._U_cache = None
        self.stats: dict = {}

    # -- factor values (device-resident after refactorize) --
    def _values(self):
        if self._host_vals is None:
            self._host_vals = self._dev.download_factors()
        return self._host_vals

    @property
    def _Lx(self):
        return self._values()[0]

    @property
    def _Ux(self):
        return self._values()[1]

    @property
    def _Udiag(self):
        return self._values()[2]

    @property
    def L(self) -> CsMatrix:
        if self._L_cache is None:
            n = self.n
            cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(self._Lp))
            idx = np.arange(n, dtype=np.int64)
            self._L_cache = from_triplets(Triplets(
                n, n, np.concatenate([self._Li, idx]), np.concatenate([cols, idx]),
                np.concatenate([self._Lx, np.ones(n)])), GENERAL)
        return self._L_cache

    @property
    def U(self) -> CsMatrix:
        if self._U_cache is None:
            n = self.n
            cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(self._Up))
            idx = np.arange(n, dtype=np.int64)
            self._U_cache = from_triplets(Triplets(
                n, n, np.concatenate([self._Ui, idx]), np.concatenate([cols, idx]),
                np.concatenate([self._Ux, self._Udiag])), GENERAL)
        return self._U_cache

    def device(self, restart_m: int = 10):
        """The device-resident system for these factors (created on first use)."""
        if self._dev is None or self._dev.h is None:  # (a closed handle is replaced)
            from .device import DeviceSystem
            self._dev = DeviceSystem(self, restart_m=restart_m)
            if self.from_refactorization and self._host_vals is not None:
                # the values of the last refactorize (kept on the host by close())
                Lx, Ux, Ud = (np.ascontiguousarray(v, dtype=np.float64) for v in self._host_vals)
                nat.check(self._dev.lib.kkt_dev_upload_factors(
                    self._dev.h, nat.ptr_f64(Lx), nat.ptr_f64(Ux), nat.ptr_f64(Ud)))
        return self._dev

    def close(self):
        """Free the device handle; the current factor values stay available on the host."""
        if self._dev is not None:
            self._values()
            self._dev.close()
            self._dev = None


def _as_general(A: CsMatrix):
    if A.symmetry == SYMMETRIC_LOWER:
        return expand_pattern(A).general
    return A


def factorize(A: CsMatrix, pivot_tol: float = 0.1):
    """Host analysis + first pivoted LU (direct_lu.py:116).  Returns (LuFactors, LuDiagnostics)."""
    if A.n_rows != A.n_cols:
        raise ValueError("factorize requires a square matrix")
    if not 0.0 < pivot_tol <= 1.0:
        raise ValueError("pivot_tol must lie in (0, 1]")
    lib = nat.load()
    Ag = _as_general(A)
    n = Ag.n_rows
    rp = np.ascontiguousarray(Ag.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(Ag.col_idx, dtype=np.int64)
    av = np.ascontiguousarray(Ag.values, dtype=np.float64)
    h = C.c_void_p()
    nat.check(lib.kkt_analyze(n, nat.ptr_i64(rp), nat.ptr_i64(ci), nat.ptr_f64(av),
                              float(pivot_tol), C.byref(h)), "kkt_analyze")
    sym = _Symbolic(h)
    sz = (C.c_int64 * 6)()
    nat.check(lib.kkt_symbolic_sizes(h, sz))
    _, _, nL, nU, nso, nap = list(sz)
    a = {k: np.empty(s, dtype=np.int64) for k, s in
         [("row_perm", n), ("col_perm", n), ("Lp", n + 1), ("Li", nL), ("Up", n + 1), ("Ui", nU),
          ("so_ptr", n + 1), ("so_data", nso), ("ap_ptr", n + 1), ("a_src", nap), ("a_tgt", nap)]}
    Lx, Ux, Ud = np.empty(nL), np.empty(nU), np.empty(n)
    I, F = nat.ptr_i64, nat.ptr_f64
    nat.check(lib.kkt_symbolic_export(
        h, I(a["row_perm"]), I(a["col_perm"]), I(a["Lp"]), I(a["Li"]), F(Lx), I(a["Up"]),
        I(a["Ui"]), F(Ux), F(Ud), I(a["so_ptr"]), I(a["so_data"]), I(a["ap_ptr"]),
        I(a["a_src"]), I(a["a_tgt"])))
    dg = (C.c_double * 4)()
    nat.check(lib.kkt_symbolic_diag(h, dg))
    st = (C.c_int64 * 9)()
    nat.check(lib.kkt_symbolic_stats(h, st))
    f = LuFactors()
    f.n = n
    f.pivot_tol = pivot_tol
    f.row_perm = Permutation(a["row_perm"])
    f.col_perm = Permutation(a["col_perm"])
    f._Lp, f._Li, f._Up, f._Ui = a["Lp"], a["Li"], a["Up"], a["Ui"]
    f._so_ptr, f._so_data = a["so_ptr"], a["so_data"]
    f._ap_ptr, f._a_src, f._a_tgt = a["ap_ptr"], a["a_src"], a["a_tgt"]
    f._host_vals = (Lx, Ux, Ud)
    f._pattern_ref = Ag
    f._sym = sym
    f.stats = dict(zip(["refactor_levels", "L_levels", "U_levels", "update_pairs", "max_so",
                        "max_L_col", "max_U_col", "max_L_row", "max_U_row"], list(st)))
    f.stats.update(nnz_L=int(nL), nnz_U=int(nU), n=int(n), nnz_general=int(Ag.nnz),
                   offdiag_pivots=int(np.count_nonzero(a["row_perm"] != a["col_perm"])),
                   refactor_flops=2 * int(st[3]) + int(nL))
    diag = LuDiagnostics(max_abs_pivot=dg[0], min_abs_pivot=dg[1],
                         zero_pivots_patched=int(dg[2]), growth_estimate=dg[3])
    return f, diag


def refactorize(factors: LuFactors, A_new: CsMatrix) -> LuDiagnostics:
    """Static-pivot numeric refactorization on the B200 (direct_lu.py:297)."""
    if not (A_new.shape == factors._pattern_ref.shape):
        raise PatternMismatchError("refactorize: sparsity pattern differs from the originally "
                                   "factorized matrix")
    dev = factors.device()
    diag = dev.refactor_matrix(A_new)
    factors.from_refactorization = True
    factors._host_vals = None
    factors._L_cache = None
    factors._U_cache = None
    return diag


def lu_solve(factors: LuFactors, b) -> np.ndarray:
    """Solve ``A x = b`` with the current factors on the device (direct_lu.py:359)."""
    b = np.asarray(b, dtype=np.float64)
    n = factors.n
    if b.shape != (n,):
        raise ValueError(f"lu_solve: b has shape {b.shape}, expected ({n},)")
    x = factors.device().solve_host(b)
    factors.triangular_solve_count += 1
    return x
