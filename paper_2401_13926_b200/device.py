"""Python owners of the device handles (``kkt_device`` / ``kkt_operator``).

PyTorch is used only as the device-memory allocator: buffers are torch tensors whose raw
pointers go through the C ABI, and all copies are issued on the library's own CUDA stream
(wrapped as a ``torch.cuda.ExternalStream``) so they order with the kernels.  There is no
CPU path: constructing a handle without a CUDA device raises.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .sparse import SYMMETRIC_LOWER, CsMatrix, lower_map


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("kktb200: no CUDA device visible; the solver path runs on the GPU "
                           "only (there is no CPU fallback)")
    return torch


def _vp(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


@dataclass
class ResidualStats:
    """Norms of e = r - K x (kkt_dev_residual_norms)."""

    err2: float
    err_inf: float
    x2: float
    x_inf: float
    r2: float
    k_inf: float

    def nsr(self) -> float:  # refine.py:62-73
        den = self.k_inf * self.x_inf
        return float("inf") if den == 0.0 else self.err_inf / den

    def nrbe(self) -> float:  # refine.py:76-85
        den = self.k_inf * self.x2 + self.r2
        return float("inf") if den == 0.0 else self.err2 / den


class DeviceSystem:
    """A factorized pattern resident on one GPU: refactor / solve / spmv / FGMRES.

    ``batch`` > 1 holds that many same-pattern systems (values, factors, vectors are
    system-major ``[batch][...]``); every call then processes all of them in one pass.
    """

    def __init__(self, factors, restart_m: int = 10, device: int = 0, batch: int = 1):
        torch = _torch()
        self.lib = nat.load()
        self.torch = torch
        self.n = factors.n
        self.nb = int(batch)
        G = factors._pattern_ref
        self.pattern = G
        lm = lower_map(G)
        self.lower = lm  # (row_ptr, col_idx, gen_src) or None (structurally unsymmetric)
        opts = nat.DeviceOpts(device=device, batch=self.nb, restart_m=int(restart_m),
                              reserved=0, flags=0)
        h = C.c_void_p()
        rp = np.ascontiguousarray(G.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(G.col_idx, dtype=np.int64)
        if lm is not None:
            gs = np.ascontiguousarray(lm[2], dtype=np.int64)
            nat.check(self.lib.kkt_dev_create(factors._sym.ptr, nat.ptr_i64(rp), nat.ptr_i64(ci),
                                              int(lm[1].size), nat.ptr_i64(gs), C.byref(opts),
                                              C.byref(h)), "kkt_dev_create")
        else:
            nat.check(self.lib.kkt_dev_create(factors._sym.ptr, nat.ptr_i64(rp), nat.ptr_i64(ci),
                                              0, None, C.byref(opts), C.byref(h)),
                      "kkt_dev_create")
        self.h = h
        self.device = torch.device("cuda", device)
        self.stream = torch.cuda.ExternalStream(self.lib.kkt_dev_stream(h), device=self.device)
        shape = (self.n,) if self.nb == 1 else (self.nb, self.n)
        f64 = torch.float64
        with torch.cuda.stream(self.stream):
            self.b = torch.empty(shape, dtype=f64, device=self.device)
            self.x = torch.empty(shape, dtype=f64, device=self.device)
            self.x0 = torch.empty(shape, dtype=f64, device=self.device)
            self.r = torch.empty(shape, dtype=f64, device=self.device)
        self._op_key = None
        self.nnz_L = int(factors._Li.size)
        self.nnz_U = int(factors._Ui.size)

    def close(self):
        if getattr(self, "h", None):
            self.lib.kkt_dev_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------- host <-> device helpers (on the library stream) ----------------
    def h2d(self, dst, a: np.ndarray):
        t = self.torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        with self.torch.cuda.stream(self.stream):
            dst.copy_(t)

    def d2h(self, src) -> np.ndarray:
        with self.torch.cuda.stream(self.stream):
            out = src.cpu()
        return out.numpy()

    def sync(self):
        self.stream.synchronize()

    # ---------------- matrix values ----------------
    def _layout_of(self, A: CsMatrix):
        if A.symmetry == SYMMETRIC_LOWER:
            if self.lower is None:
                raise ValueError("symmetric-lower values for a structurally unsymmetric pattern")
            if not (np.array_equal(A.row_ptr, self.lower[0])
                    and np.array_equal(A.col_idx, self.lower[1])):
                from .direct_lu import PatternMismatchError
                raise PatternMismatchError("refactorize: sparsity pattern differs from the "
                                           "originally factorized matrix")
            return nat.LAYOUT_SYMMETRIC_LOWER
        if not A.same_pattern(self.pattern):
            from .direct_lu import PatternMismatchError
            raise PatternMismatchError("refactorize: sparsity pattern differs from the "
                                       "originally factorized matrix")
        return nat.LAYOUT_GENERAL

    def refactor_matrix(self, A: CsMatrix):
        from .direct_lu import LuDiagnostics
        layout = self._layout_of(A)
        vals = np.ascontiguousarray(A.values, dtype=np.float64)
        dg = (C.c_double * 4)()
        nat.check(self.lib.kkt_dev_refactor(self.h, vals.ctypes.data_as(C.c_void_p), layout, 0, dg),
                  "kkt_dev_refactor")
        self._op_key = (id(A.values), layout)
        self._op_ref = A.values
        return LuDiagnostics(max_abs_pivot=dg[0], min_abs_pivot=dg[1],
                             zero_pivots_patched=int(dg[2]), growth_estimate=dg[3])

    def refactor_device(self, values_t, layout: int):
        """Refactorize from device-resident values (no host traffic, no sync)."""
        nat.check(self.lib.kkt_dev_refactor(self.h, _vp(values_t), layout, 1, None),
                  "kkt_dev_refactor")
        self._op_key = None

    def set_operator(self, K: CsMatrix):
        """Make K the FGMRES / spmv operator (skips the upload when it is already current)."""
        layout = self._layout_of(K)
        key = (id(K.values), layout)
        vals = np.ascontiguousarray(K.values, dtype=np.float64)
        nat.check(self.lib.kkt_dev_set_operator_values(self.h, vals.ctypes.data_as(C.c_void_p),
                                                       layout, 0), "set_operator_values")
        self._op_key = key
        self._op_ref = K.values

    def download_factors(self):
        Lx, Ux, Ud = np.empty(self.nnz_L), np.empty(self.nnz_U), np.empty(self.n)
        nat.check(self.lib.kkt_dev_download_factors(self.h, nat.ptr_f64(Lx), nat.ptr_f64(Ux),
                                                    nat.ptr_f64(Ud)))
        return Lx, Ux, Ud

    # ---------------- kernels ----------------
    def solve_device(self, b_t, x_t):
        nat.check(self.lib.kkt_dev_solve(self.h, _vp(b_t), _vp(x_t)), "kkt_dev_solve")

    def solve_host(self, b: np.ndarray) -> np.ndarray:
        self.h2d(self.b, b)
        self.solve_device(self.b, self.x)
        return self.d2h(self.x)

    def nbp(self) -> int:
        """interleaved width of the handle's internal vectors (1 for a single system)"""
        return 1 if self.nb == 1 else (self.nb + 31) // 32 * 32

    def solve_native(self, b_t, x_t):
        """lu_solve kernels on internal-layout vectors ([n][nbp]; no boundary transposes)"""
        nat.check(self.lib.kkt_dev_solve_native(self.h, _vp(b_t), _vp(x_t)), "kkt_dev_solve_native")

    def spmv_native(self, x_t, y_t):
        """SpMV kernel on internal-layout vectors ([n][nbp]; no boundary transposes)"""
        nat.check(self.lib.kkt_dev_spmv_native(self.h, _vp(x_t), _vp(y_t)), "kkt_dev_spmv_native")

    def spmv_device(self, x_t, y_t):
        nat.check(self.lib.kkt_dev_spmv(self.h, _vp(x_t), _vp(y_t)), "kkt_dev_spmv")

    def residual_device(self, r_t, x_t, rho_t):
        """rho = r - K x (reference spmv order) and ||rho||_2 per system (kkt_dev_residual)."""
        out = (C.c_double * self.nb)()
        nat.check(self.lib.kkt_dev_residual(self.h, _vp(r_t), _vp(x_t), _vp(rho_t), out),
                  "kkt_dev_residual")
        return out[0] if self.nb == 1 else list(out)

    def axpy_device(self, x_t, y_t):
        """x += y on the device (kkt_dev_axpy)."""
        nat.check(self.lib.kkt_dev_axpy(self.h, _vp(x_t), _vp(y_t)), "kkt_dev_axpy")

    def residual_stats_device(self, r_t, x_t):
        """ResidualStats of r - K x (one per system on a batched handle)."""
        out = (C.c_double * (6 * self.nb))()
        nat.check(self.lib.kkt_dev_residual_norms(self.h, _vp(r_t), _vp(x_t), out))
        stats = [ResidualStats(*out[6 * q:6 * q + 6]) for q in range(self.nb)]
        return stats[0] if self.nb == 1 else stats

    def fgmres_device(self, b_t, x0_t, x_t, m: int, max_outer: int, tol: float,
                      K=None, M=None, host_loop: bool = False, flags: int = 0):
        """FGMRES (krylov.py:117) on every system: returns (report, history, restart_pairs)
        or a list of them (batch).  K / M: ``nat.LinOp`` (None = the handle's operator values /
        LU factors).  The whole solve is one device-controlled CUDA graph unless a host
        callback operator (or ``host_loop``) asks for the host-stepped control."""
        cfg = nat.KrylovCfg(m=int(m), max_outer=int(max_outer), tol=float(tol), delta_tol=float(tol),
                            flags=flags | (nat.FG_HOST_LOOP if host_loop else 0))
        reps = (nat.KrylovReport * self.nb)()
        hcap = int(max_outer) * int(m) + 1
        pcap = max(int(max_outer), 1)
        hist = (C.c_double * (hcap * self.nb))()
        pairs = (C.c_double * (2 * pcap * self.nb))()
        rc = self.lib.kkt_dev_fgmres_ops(self.h, C.byref(K) if K is not None else None,
                                         C.byref(M) if M is not None else None, _vp(b_t), _vp(x0_t),
                                         _vp(x_t), C.byref(cfg), reps, hist, hcap, pairs, pcap)
        nat.check(rc, "kkt_dev_fgmres_ops")
        out = []
        for q in range(self.nb):
            nh = min(reps[q].iterations + 1, hcap)
            npair = min(reps[q].restarts, pcap)
            out.append((reps[q], [hist[q * hcap + i] for i in range(nh)],
                        [(pairs[2 * (q * pcap + i)], pairs[2 * (q * pcap + i) + 1])
                         for i in range(npair)]))
        return out[0] if self.nb == 1 else out

    def refine_device(self, r_t, x0_t, x_t, m: int, max_outer: int, delta_tol,
                      host_loop: bool = False, mgs: bool = False):
        """refine_fgmres (refine.py:103-132) in one call: trigger, FGMRES and the residual
        statistics before / after, decided on the device; one host synchronisation."""
        dsys = None
        if np.ndim(delta_tol):
            dsys = (C.c_double * self.nb)(*[float(v) for v in delta_tol])
            delta_tol = float(np.max(delta_tol))
        flags = (nat.FG_STATS_AFTER | (nat.FG_HOST_LOOP if host_loop else 0)
                 | (nat.FG_MGS if mgs else 0))
        cfg = nat.KrylovCfg(m=int(m), max_outer=int(max_outer), tol=float(delta_tol),
                            delta_tol=float(delta_tol), delta_sys=dsys, flags=flags)
        reps = (nat.KrylovReport * self.nb)()
        rc = self.lib.kkt_dev_refine_fgmres(self.h, _vp(r_t), _vp(x0_t), _vp(x_t), C.byref(cfg), reps)
        self._check_batch(rc, "kkt_dev_refine_fgmres")
        return reps[0] if self.nb == 1 else list(reps)

    def _check_batch(self, rc, what):
        # a batch reports non-finite failures per system (KrylovReport.nonfinite) and still
        # returns every other system's solution; a single system raises like the reference
        if rc == nat.KKT_ERR_NONFINITE and self.nb > 1:
            return
        nat.check(rc, what)

    def step(self, values: np.ndarray | object, layout: int, r, x_out, on_device: bool,
             m: int, max_outer: int, delta_tol, diag: bool = False, stats: bool = False,
             handoff: bool = True):
        """refactor -> solve -> refine_fgmres in one C call (kkt_dev_step) for every system.

        ``delta_tol`` is a float or a per-system sequence.  Returns the KrylovReport (single
        system) or the list of reports (batch); with ``diag`` also the per-system
        LuDiagnostics array ``[nb][4]``.  ``stats`` also fills the reports' residual statistics
        of x0 and x (nsr / nrbe before and after, refine.py:117,129-131).  ``handoff``
        (batched handles): the last few running systems finish on single-system helpers
        (KrylovReport.handed_off) instead of in the lockstep batch.
        """
        dsys = None
        if np.ndim(delta_tol):
            dsys = (C.c_double * self.nb)(*[float(v) for v in delta_tol])
            delta_tol = float(np.max(delta_tol))
        cfg = nat.KrylovCfg(m=int(m), max_outer=int(max_outer), tol=float(delta_tol),
                            delta_tol=float(delta_tol), delta_sys=dsys,
                            flags=(nat.FG_STATS_AFTER if stats else 0)
                            | (0 if handoff else nat.FG_NO_HANDOFF))
        reps = (nat.KrylovReport * self.nb)()
        dg = (C.c_double * (4 * self.nb))() if diag else None
        if on_device:
            args = (_vp(values), layout, _vp(r), _vp(x_out), 1)
        else:
            args = (values.ctypes.data_as(C.c_void_p), layout, r.ctypes.data_as(C.c_void_p),
                    x_out.ctypes.data_as(C.c_void_p), 0)
        self._check_batch(self.lib.kkt_dev_step(self.h, *args, C.byref(cfg), reps, dg), "kkt_dev_step")
        self._op_key = None
        rep = reps[0] if self.nb == 1 else list(reps)
        if diag:
            return rep, np.array(list(dg)).reshape(self.nb, 4)
        return rep

    def step_solve(self, r, x_out, on_device: bool, m: int, max_outer: int, delta_tol):
        """solve -> refine_fgmres for the factors of the last refactor (kkt_dev_step_solve):
        the second half of ``step``, so the rhs upload can overlap the refactorization."""
        dsys = None
        if np.ndim(delta_tol):
            dsys = (C.c_double * self.nb)(*[float(v) for v in delta_tol])
            delta_tol = float(np.max(delta_tol))
        cfg = nat.KrylovCfg(m=int(m), max_outer=int(max_outer), tol=float(delta_tol),
                            delta_tol=float(delta_tol), delta_sys=dsys)
        reps = (nat.KrylovReport * self.nb)()
        if on_device:
            args = (_vp(r), _vp(x_out), 1)
        else:
            args = (r.ctypes.data_as(C.c_void_p), x_out.ctypes.data_as(C.c_void_p), 0)
        self._check_batch(self.lib.kkt_dev_step_solve(self.h, *args, C.byref(cfg), reps),
                          "kkt_dev_step_solve")
        return reps[0] if self.nb == 1 else list(reps)

    def refactor_batch(self, values_t, layout: int) -> np.ndarray:
        """Refactorize all systems from device values [nb][nnz]; returns diagnostics [nb][4]."""
        dg = (C.c_double * (4 * self.nb))()
        nat.check(self.lib.kkt_dev_refactor(self.h, _vp(values_t), layout, 1, dg), "kkt_dev_refactor")
        self._op_key = None
        return np.array(list(dg)).reshape(self.nb, 4)

    def download_factors_batch(self):
        Lx = np.empty(self.nnz_L * self.nb)
        Ux = np.empty(self.nnz_U * self.nb)
        Ud = np.empty(self.n * self.nb)
        nat.check(self.lib.kkt_dev_download_factors(self.h, nat.ptr_f64(Lx), nat.ptr_f64(Ux),
                                                    nat.ptr_f64(Ud)))
        return (Lx.reshape(self.nb, -1), Ux.reshape(self.nb, -1), Ud.reshape(self.nb, -1))

    def info(self) -> dict:
        v = (C.c_int64 * 16)()
        nat.check(self.lib.kkt_dev_info(self.h, v))
        keys = ["n", "pL", "pU", "L_grid_levels", "U_grid_levels", "L_tail_rows", "U_head_rows",
                "refactor_blocks", "refactor_warps", "refactor_smem", "trsv_blocks",
                "refactor_levels", "arena_bytes", "update_pairs"]
        return {k: int(v[i]) for i, k in enumerate(keys)}

    def launch_count(self) -> int:
        return int(self.lib.kkt_dev_launch_count(self.h))


class DeviceOperator:
    """A bare matrix on the device (sparsecore.spmv / nsr / nrbe without factors)."""

    def __init__(self, A: CsMatrix, device: int = 0):
        torch = _torch()
        self.torch = torch
        self.lib = nat.load()
        self.n = A.n_rows
        if A.n_rows != A.n_cols:
            raise ValueError("operator matrices must be square")
        rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.col_idx, dtype=np.int64)
        h = C.c_void_p()
        nat.check(self.lib.kkt_op_create(A.n_rows, nat.ptr_i64(rp), nat.ptr_i64(ci),
                                         1 if A.symmetry == SYMMETRIC_LOWER else 0, device,
                                         C.byref(h)), "kkt_op_create")
        self.h = h
        self.pattern = (A.row_ptr, A.col_idx, A.symmetry)
        self.device = torch.device("cuda", device)
        self.stream = torch.cuda.ExternalStream(self.lib.kkt_op_stream(h), device=self.device)
        with torch.cuda.stream(self.stream):
            self.a = torch.empty(self.n, dtype=torch.float64, device=self.device)
            self.b = torch.empty(self.n, dtype=torch.float64, device=self.device)
        self._vals_ref = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.kkt_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_values(self, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.float64)
        nat.check(self.lib.kkt_op_set_values(self.h, v.ctypes.data_as(C.c_void_p), 0))
        self._vals_ref = values

    def _h2d(self, dst, a):
        with self.torch.cuda.stream(self.stream):
            dst.copy_(self.torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)))

    def spmv(self, x: np.ndarray) -> np.ndarray:
        self._h2d(self.a, x)
        nat.check(self.lib.kkt_op_spmv(self.h, _vp(self.a), _vp(self.b)))
        with self.torch.cuda.stream(self.stream):
            return self.b.cpu().numpy()

    def residual_stats(self, r: np.ndarray, x: np.ndarray) -> ResidualStats:
        self._h2d(self.a, r)
        self._h2d(self.b, x)
        out = (C.c_double * 6)()
        nat.check(self.lib.kkt_op_residual_norms(self.h, _vp(self.a), _vp(self.b), out))
        return ResidualStats(*list(out))


_OPS: dict = {}


def operator_for(A: CsMatrix) -> DeviceOperator:
    """Device operator cached per pattern object (values refreshed on identity change)."""
    key = (id(A.row_ptr), id(A.col_idx), A.symmetry)
    op = _OPS.get(key)
    if op is None or op.pattern[0] is not A.row_ptr:
        if len(_OPS) > 16:
            for k in list(_OPS)[:8]:
                _OPS.pop(k).close()
        op = DeviceOperator(A)
        _OPS[key] = op
    op.set_values(A.values)
    return op
