"""Drop-in for ``kktsolve.krylov``: restarted FGMRES(m) + CGS2 (or MGS) on the B200.

The device FGMRES (``kkt_dev_fgmres_ops``) runs the Arnoldi step as fused multi-dot /
multi-axpy kernels and the Hessenberg/Givens update, the stop tests and the restart logic as
device control kernels (krylov.py:117-208): one CUDA graph per solve, one host sync.
Operators are the reference's ``LinearOperator`` (krylov.py:36-54):

* ``LinearOperator.from_matrix(A)``: device SpMV (the factors' handle when A has their
  pattern, else a standalone device operator);
* ``LinearOperator.identity(n)``: device copy;
* :func:`lu_preconditioner` ``(factors)``: the device triangular solves;
* any other ``LinearOperator(n, apply)``: the user's host callback, called on numpy vectors
  exactly like the reference (the iteration's other work stays on the device; the control
  then steps from the host because a Python callback cannot run inside a CUDA graph).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

CGS2 = "cgs2"
MGS = "mgs"
HAPPY_BREAKDOWN_RTOL = 1e-14  # krylov.py:25


class OperatorOutputError(RuntimeError):
    """An operator produced a NaN or Inf entry (krylov.py:28)."""


class NotSpdOperatorError(RuntimeError):
    """CG observed p.S.p <= 0 (krylov.py:32); CG is outside the hot path."""


@dataclass
class LinearOperator:
    """Square operator: dimension + apply callback (krylov.py:36-54).

    ``matrix`` / ``factors`` / ``is_identity`` mark the device-backed kinds; ``apply`` is
    the reference's callback (a host function of numpy vectors) for every other operator.
    """

    dimension: int
    apply: Callable[[np.ndarray], np.ndarray]
    matrix: object = None
    factors: object = None
    is_identity: bool = False

    def __call__(self, v: np.ndarray) -> np.ndarray:
        return self.apply(v)

    @classmethod
    def from_matrix(cls, A) -> "LinearOperator":
        if A.n_rows != A.n_cols:
            raise ValueError("operator matrices must be square")
        from .sparse_ops import spmv
        return cls(A.n_rows, lambda v: spmv(A, v), matrix=A)

    @classmethod
    def identity(cls, n: int) -> "LinearOperator":
        op = cls(n, lambda v: np.asarray(v, dtype=np.float64).copy())
        op.is_identity = True
        return op


def lu_preconditioner(factors) -> LinearOperator:
    """M(v) = lu_solve(factors, v) as a device-backed operator (refine.py:119)."""
    from .direct_lu import lu_solve
    return LinearOperator(factors.n, lambda v: lu_solve(factors, v), factors=factors)


@dataclass
class KrylovConfig:
    """Restart length, restart-cycle budget, tolerance (krylov.py:57-72)."""

    m: int = 10
    max_outer: int = 10
    tol: float = 1e-12
    ortho: str = CGS2

    def __post_init__(self):
        if self.m < 1:
            raise ValueError("restart length m must be >= 1")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.ortho not in (CGS2, MGS):
            raise ValueError(f"unknown orthogonalization {self.ortho!r}")


@dataclass
class KrylovResult:
    x: np.ndarray
    iterations: int
    converged: bool
    est_residual_history: list
    true_final_residual: float
    precond_applications: int
    restart_residuals: list = field(default_factory=list)


def _matrix_of(op):
    return getattr(op, "matrix", None)


def _factors_of(op):
    return getattr(op, "factors", None)


_WORKSPACES: dict = {}


def _workspace_device(n: int):
    """A device handle that only provides the FGMRES workspace (no factors are used): the
    analysis of the n x n identity, cached per n."""
    dev = _WORKSPACES.get(n)
    if dev is None:
        from .direct_lu import factorize
        from .sparse import GENERAL, CsMatrix
        idx = np.arange(n, dtype=np.int64)
        eye = CsMatrix(n, n, np.arange(n + 1, dtype=np.int64), idx, np.ones(n), GENERAL)
        f, _ = factorize(eye)
        dev = f.device()
        dev._owner = f
        _WORKSPACES[n] = dev
    return dev


def fgmres(K: LinearOperator, M: LinearOperator, b, x0, cfg: KrylovConfig) -> KrylovResult:
    """Right-preconditioned flexible GMRES(m) on the device (krylov.py:117-208)."""
    import ctypes as C

    from . import _native as nat
    from .device import operator_for
    n = K.dimension
    b = np.asarray(b, dtype=np.float64)
    x0 = np.asarray(x0, dtype=np.float64)
    if b.shape != (n,) or x0.shape != (n,):
        raise ValueError("fgmres: dimension mismatch")
    factors = _factors_of(M)
    A = _matrix_of(K)
    if factors is not None and factors.n == n:
        dev = factors.device(restart_m=cfg.m)
    else:
        factors = None
        dev = _workspace_device(n)
    keep = []  # ctypes callbacks and operators alive for the duration of the call

    def linop_K():
        if A is not None:
            if factors is not None:
                try:
                    dev.set_operator(A)
                    return None  # the handle's own operator values
                except Exception:
                    pass
            op = operator_for(A)
            keep.append(op)
            return nat.LinOp(kind=nat.OP_MATRIX, matrix=op.h)
        if getattr(K, "is_identity", False):
            return nat.LinOp(kind=nat.OP_IDENTITY)
        return _callback_op(K, n, keep)

    def linop_M():
        if factors is not None:
            return None  # the handle's LU factors
        if getattr(M, "is_identity", False):
            return nat.LinOp(kind=nat.OP_IDENTITY)
        Am = _matrix_of(M)
        if Am is not None:
            op = operator_for(Am)
            keep.append(op)
            return nat.LinOp(kind=nat.OP_MATRIX, matrix=op.h)
        return _callback_op(M, n, keep)

    lk, lm = linop_K(), linop_M()
    host = any(isinstance(o, nat.LinOp) and o.kind == nat.OP_CALLBACK for o in (lk, lm))
    dev.h2d(dev.b, b)
    dev.h2d(dev.x0, x0)
    flags = nat.FG_MGS if cfg.ortho == MGS else 0
    try:
        rep, hist, pairs = dev.fgmres_device(dev.b, dev.x0, dev.x, cfg.m, cfg.max_outer, cfg.tol,
                                             K=lk, M=lm, host_loop=host, flags=flags)
    except RuntimeError as exc:
        for err in keep:
            if isinstance(err, BaseException):
                raise err from exc
        raise
    if factors is not None and lm is None:
        factors.triangular_solve_count += rep.precond_applications
    x = dev.d2h(dev.x)
    return KrylovResult(x=x, iterations=rep.iterations, converged=bool(rep.converged),
                        est_residual_history=hist, true_final_residual=rep.true_final,
                        precond_applications=rep.precond_applications,
                        restart_residuals=pairs)


def _callback_op(L: LinearOperator, n: int, keep: list):
    """A host callback operator: the C library hands over pinned numpy-visible buffers."""
    import ctypes as C

    from . import _native as nat

    def apply(_user, pin, pout):
        try:
            v = np.ctypeslib.as_array(C.cast(pin, C.POINTER(C.c_double)), shape=(n,)).copy()
            y = np.asarray(L.apply(v), dtype=np.float64)
            if y.shape != (n,):
                raise ValueError("fgmres: operator returned the wrong shape")
            np.ctypeslib.as_array(C.cast(pout, C.POINTER(C.c_double)), shape=(n,))[:] = y
            return 0
        except BaseException as exc:  # re-raised after the C call returns
            keep.append(exc)
            return 1

    fn = nat.APPLY_FN(apply)
    keep.append(fn)
    return nat.LinOp(kind=nat.OP_CALLBACK, apply=fn)
