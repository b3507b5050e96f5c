"""Drop-in for ``kktsolve.krylov``: restarted FGMRES(m) + CGS2 on the B200.

The device FGMRES (``kkt_dev_fgmres``) applies K as the device SpMV of a matrix and M as the
device LU triangular solves; the Arnoldi CGS2 step runs as fused multi-dot / multi-axpy
kernels and the Hessenberg/Givens update as an on-device kernel (krylov.py:117-208).
Operators are expressed with the reference's ``LinearOperator`` type:
``LinearOperator.from_matrix(K)`` and :func:`lu_preconditioner` ``(factors)`` are the two
device-backed operators; an arbitrary Python callback has no device implementation and is
rejected (there is no CPU fallback).
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

    ``matrix`` / ``factors`` mark the two device-backed kinds; ``apply`` is kept for API
    parity and evaluates through the device too.
    """

    dimension: int
    apply: Callable[[np.ndarray], np.ndarray]
    matrix: object = None
    factors: object = None

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
        return cls(n, lambda v: np.asarray(v, dtype=np.float64).copy())


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


def fgmres(K: LinearOperator, M: LinearOperator, b, x0, cfg: KrylovConfig) -> KrylovResult:
    """Right-preconditioned flexible GMRES(m) on the device (krylov.py:117)."""
    n = K.dimension
    b = np.asarray(b, dtype=np.float64)
    x0 = np.asarray(x0, dtype=np.float64)
    if b.shape != (n,) or x0.shape != (n,):
        raise ValueError("fgmres: dimension mismatch")
    if K.matrix is None or M.factors is None:
        raise TypeError("fgmres on the B200 needs K = LinearOperator.from_matrix(A) and "
                        "M = lu_preconditioner(factors); arbitrary callbacks have no device path")
    if cfg.ortho != CGS2:
        raise NotImplementedError("the device Arnoldi step implements CGS2 (the hot-path "
                                  "default); MGS is not provided")
    factors = M.factors
    dev = factors.device(restart_m=cfg.m)
    dev.set_operator(K.matrix)
    dev.h2d(dev.b, b)
    dev.h2d(dev.x0, x0)
    rep, hist = dev.fgmres_device(dev.b, dev.x0, dev.x, cfg.m, cfg.max_outer, cfg.tol)
    factors.triangular_solve_count += rep.precond_applications
    x = dev.d2h(dev.x)
    return KrylovResult(x=x, iterations=rep.iterations, converged=bool(rep.converged),
                        est_residual_history=hist, true_final_residual=rep.true_final,
                        precond_applications=rep.precond_applications,
                        restart_residuals=[])
