"""Device-backed sparse kernels with the reference's host signatures.

``spmv`` (sparsecore.py:284) and ``inf_norm`` (sparsecore.py:333) for a bare matrix run on
the GPU through a cached ``kkt_operator`` handle, in the reference's accumulation order.
"""

from __future__ import annotations

import numpy as np

from .sparse import CsMatrix, SparseError


def spmv(A: CsMatrix, x, transpose: bool = False) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    need = A.n_rows if transpose else A.n_cols
    if x.shape != (need,):
        raise SparseError(f"spmv: x has length {x.shape}, expected ({need},)")
    if transpose and A.symmetry != "symmetric-lower":
        raise NotImplementedError("transposed spmv of a general matrix is not on the hot path")
    from .device import operator_for
    return operator_for(A).spmv(x)


def residual_stats(A: CsMatrix, r, x):
    """Norms of r - A x plus ||A||_inf (one device pass)."""
    from .device import operator_for
    return operator_for(A).residual_stats(np.asarray(r, dtype=np.float64),
                                          np.asarray(x, dtype=np.float64))


def inf_norm(A: CsMatrix) -> float:
    if A.nnz == 0:
        return 0.0
    n = A.n_rows
    return residual_stats(A, np.zeros(n), np.zeros(n)).k_inf
