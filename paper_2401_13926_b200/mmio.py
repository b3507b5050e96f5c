"""Drop-in for ``kktsolve.mmio``: Matrix Market readers in C++ (SURVEY.md §8f row 4), writers
as the reference's (17 significant digits, so a write/read round trip is exact).

``load_matrix_market`` / ``load_vector`` parse through ``kkt_mm_*`` (libkktb200.so) — same
dialect, same checks, same "path:line: message" errors as mmio.py:36-130 — and build the
CsMatrix with ``from_triplets`` exactly like the reference.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .sparse import GENERAL, SYMMETRIC_LOWER, CsMatrix, Triplets, from_triplets


class MatrixMarketError(ValueError):
    """Malformed Matrix Market content; message includes the line number (mmio.py:17)."""


def _check(rc):
    if rc != 0:
        raise MatrixMarketError(nat.last_error())


def _info(path: str):
    info = np.zeros(5, dtype=np.int64)
    _check(nat.load().kkt_mm_info(str(path).encode(), nat.ptr_i64(info)))
    return info


def load_matrix_market(path: str) -> CsMatrix:
    """Coordinate real general/symmetric file -> CsMatrix (mmio.py:36-93)."""
    fmt, sym, n_rows, n_cols, nnz = (int(v) for v in _info(path))
    if fmt != 0:
        raise MatrixMarketError(f"{path}:1: expected a coordinate matrix, got 'array'")
    rows = np.empty(nnz, dtype=np.int64)
    cols = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz, dtype=np.float64)
    _check(nat.load().kkt_mm_read_coo(str(path).encode(), nnz, nat.ptr_i64(rows), nat.ptr_i64(cols),
                                      nat.ptr_f64(vals)))
    tag = SYMMETRIC_LOWER if sym else GENERAL
    return from_triplets(Triplets(n_rows, n_cols, rows, cols, vals), tag)


def load_vector(path: str) -> np.ndarray:
    """Array real file (or an n x 1 coordinate file) -> vector (mmio.py:96-130)."""
    fmt, _sym, n_rows, n_cols, _nnz = (int(v) for v in _info(path))
    if fmt == 0:
        A = load_matrix_market(path)
        if A.n_cols != 1:
            raise MatrixMarketError(f"{path}: expected a single-column vector")
        out = np.zeros(A.n_rows)
        rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
        out[rows] = A.values
        return out
    out = np.empty(n_rows)
    _check(nat.load().kkt_mm_read_array(str(path).encode(), n_rows, nat.ptr_f64(out)))
    return out


def write_matrix_market(path: str, A: CsMatrix) -> None:
    """CSR content as coordinate real general/symmetric, 1-based (mmio.py:137-145)."""
    sym = "symmetric" if A.symmetry == SYMMETRIC_LOWER else "general"
    rows = np.repeat(np.arange(A.n_rows, dtype=np.int64), np.diff(A.row_ptr))
    with open(path, "w") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate real {sym}\n")
        fh.write(f"{A.n_rows} {A.n_cols} {A.nnz}\n")
        fh.writelines(f"{r + 1} {c + 1} {v:.17g}\n" for r, c, v in zip(rows, A.col_idx, A.values))


def write_vector(path: str, v) -> None:
    """A vector as matrix array real general, n x 1 (mmio.py:148-155)."""
    v = np.asarray(v, dtype=np.float64)
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix array real general\n")
        fh.write(f"{v.size} 1\n")
        fh.writelines(f"{x:.17g}\n" for x in v)
