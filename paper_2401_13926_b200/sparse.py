"""Host-side sparse pattern storage: the reference's ``CsMatrix`` contract.

Mirrors ``kktsolve.sparsecore`` (sparsecore.py:52-273) closely enough that the
reference's harness and tests can hand their matrices to this package unchanged:
CSR with int64 ``row_ptr``/``col_idx`` (sorted, unique per row), float64 ``values``,
``symmetry`` in {"general", "symmetric-lower"}, write-protected pattern arrays.

Only integer pattern plumbing lives here (expansion of symmetric-lower storage into the
general pattern, transposition maps).  Every floating-point kernel of the hot path runs
on the GPU through ``libkktb200.so``; nothing here computes matrix-vector products.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GENERAL = "general"
SYMMETRIC_LOWER = "symmetric-lower"


class SparseError(ValueError):
    """Structural problems: bad indices, shape mismatch (sparsecore.py:21)."""


@dataclass
class Triplets:
    """Coordinate entries; duplicates are summed by :func:`from_triplets`."""

    n_rows: int
    n_cols: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    @classmethod
    def from_entries(cls, n_rows: int, n_cols: int, entries) -> "Triplets":
        ent = list(entries)
        r = np.array([e[0] for e in ent], dtype=np.int64)
        c = np.array([e[1] for e in ent], dtype=np.int64)
        v = np.array([e[2] for e in ent], dtype=np.float64)
        return cls(n_rows, n_cols, r, c, v)


@dataclass
class Permutation:
    """``perm[new] = old``, ``inv_perm[old] = new`` (sparsecore.py:52-79)."""

    perm: np.ndarray
    inv_perm: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self):
        self.perm = np.asarray(self.perm, dtype=np.int64)
        n = self.perm.size
        if n:
            seen = np.zeros(n, dtype=np.int64)
            ok = self.perm.min() >= 0 and self.perm.max() < n
            if ok:
                np.add.at(seen, self.perm, 1)
            if not ok or np.any(seen != 1):
                raise SparseError("permutation is not a bijection")
        if self.inv_perm is None:
            inv = np.empty(n, dtype=np.int64)
            inv[self.perm] = np.arange(n, dtype=np.int64)
            self.inv_perm = inv

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        return cls(np.arange(n, dtype=np.int64))

    def inverse(self) -> "Permutation":
        return Permutation(self.inv_perm.copy(), self.perm.copy())

    @property
    def n(self) -> int:
        return int(self.perm.size)


class CsMatrix:
    """CSR with a frozen pattern (sparsecore.py:91-213)."""

    __slots__ = ("n_rows", "n_cols", "row_ptr", "col_idx", "values", "symmetry",
                 "_row_of_entry")

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values, symmetry=GENERAL,
                 _checked=False):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(col_idx, dtype=np.int64)
        self.values = np.asarray(values, dtype=np.float64)
        self.symmetry = symmetry
        self._row_of_entry = None
        if not _checked:
            self._validate()
        self.row_ptr.flags.writeable = False
        self.col_idx.flags.writeable = False

    def _validate(self):
        if self.symmetry not in (GENERAL, SYMMETRIC_LOWER):
            raise SparseError(f"unknown symmetry tag {self.symmetry!r}")
        if self.symmetry == SYMMETRIC_LOWER and self.n_rows != self.n_cols:
            raise SparseError("symmetric storage requires a square matrix")
        if self.row_ptr.size != self.n_rows + 1:
            raise SparseError("row_ptr has wrong length")
        if self.row_ptr[0] != 0 or self.row_ptr[-1] != self.col_idx.size:
            raise SparseError("row_ptr endpoints inconsistent with nnz")
        d = np.diff(self.row_ptr)
        if np.any(d < 0):
            raise SparseError("row_ptr must be nondecreasing")
        if self.col_idx.size != self.values.size:
            raise SparseError("col_idx and values lengths differ")
        if self.col_idx.size == 0:
            return
        if self.col_idx.min() < 0 or self.col_idx.max() >= self.n_cols:
            raise SparseError("column index out of range")
        rows = np.repeat(np.arange(self.n_rows, dtype=np.int64), d)
        same_row = rows[1:] == rows[:-1]
        bad = same_row & (self.col_idx[1:] <= self.col_idx[:-1])
        if np.any(bad):
            i = int(rows[1:][bad][0])
            raise SparseError(f"row {i}: column indices not strictly increasing")
        if self.symmetry == SYMMETRIC_LOWER and np.any(self.col_idx > rows):
            i = int(rows[self.col_idx > rows][0])
            raise SparseError(f"row {i}: entry above diagonal in symmetric-lower storage")

    @property
    def nnz(self) -> int:
        return int(self.col_idx.size)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def row_of_entry(self) -> np.ndarray:
        if self._row_of_entry is None:
            r = np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.row_ptr))
            r.flags.writeable = False
            self._row_of_entry = r
        return self._row_of_entry

    def set_values(self, new_values) -> None:
        new_values = np.asarray(new_values, dtype=np.float64)
        if new_values.size != self.values.size:
            raise SparseError("value array length does not match pattern nnz")
        self.values[:] = new_values

    def _share(self, values) -> "CsMatrix":
        out = CsMatrix.__new__(CsMatrix)
        out.n_rows, out.n_cols = self.n_rows, self.n_cols
        out.row_ptr, out.col_idx = self.row_ptr, self.col_idx
        out.values = values
        out.symmetry = self.symmetry
        out._row_of_entry = self._row_of_entry
        return out

    def copy(self, share_pattern: bool = True) -> "CsMatrix":
        if share_pattern:
            return self._share(self.values.copy())
        return CsMatrix(self.n_rows, self.n_cols, self.row_ptr.copy(), self.col_idx.copy(),
                        self.values.copy(), self.symmetry)

    def same_pattern(self, other) -> bool:
        if self.shape != tuple(other.shape):
            return False
        if self.row_ptr is other.row_ptr and self.col_idx is other.col_idx:
            return True
        return (np.array_equal(self.row_ptr, other.row_ptr)
                and np.array_equal(self.col_idx, other.col_idx))

    def with_values(self, values) -> "CsMatrix":
        values = np.asarray(values, dtype=np.float64)
        if values.size != self.nnz:
            raise SparseError("value array length does not match pattern nnz")
        return self._share(values)

    def to_dense(self) -> np.ndarray:
        M = np.zeros((self.n_rows, self.n_cols))
        rows = self.row_of_entry()
        M[rows, self.col_idx] = self.values
        if self.symmetry == SYMMETRIC_LOWER:
            s = rows != self.col_idx
            M[self.col_idx[s], rows[s]] = self.values[s]
        return M

    def __repr__(self):
        return f"CsMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz}, {self.symmetry})"


def from_triplets(t: Triplets, symmetry: str = GENERAL) -> CsMatrix:
    """Sorted CSR from coordinates, duplicates summed in input order (sparsecore.py:216)."""
    rows = np.asarray(t.rows, dtype=np.int64)
    cols = np.asarray(t.cols, dtype=np.int64)
    vals = np.asarray(t.values, dtype=np.float64)
    if rows.size and (rows.min() < 0 or rows.max() >= t.n_rows):
        raise SparseError("row index out of range")
    if cols.size and (cols.min() < 0 or cols.max() >= t.n_cols):
        raise SparseError("column index out of range")
    key = np.lexsort((cols, rows))
    rows, cols, vals = rows[key], cols[key], vals[key]
    if rows.size:
        head = np.ones(rows.size, dtype=bool)
        head[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        starts = np.flatnonzero(head)
        urows, ucols = rows[starts], cols[starts]
        uvals = np.add.reduceat(vals, starts)
    else:
        urows = ucols = np.empty(0, dtype=np.int64)
        uvals = np.empty(0)
    row_ptr = np.zeros(t.n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(urows, minlength=t.n_rows), out=row_ptr[1:])
    return CsMatrix(t.n_rows, t.n_cols, row_ptr, ucols, uvals, symmetry, _checked=True)


def from_dense(M, symmetry: str = GENERAL, drop_tol: float = 0.0) -> CsMatrix:
    M = np.asarray(M, dtype=np.float64)
    keep = np.abs(M) > drop_tol
    if symmetry == SYMMETRIC_LOWER:
        keep &= np.tril(np.ones_like(keep, dtype=bool))
    r, c = np.nonzero(keep)
    return from_triplets(Triplets(M.shape[0], M.shape[1], r.astype(np.int64),
                                  c.astype(np.int64), M[r, c]), symmetry)


def identity(n: int) -> CsMatrix:
    idx = np.arange(n, dtype=np.int64)
    return CsMatrix(n, n, np.arange(n + 1, dtype=np.int64), idx, np.ones(n), _checked=True)


@dataclass
class Expansion:
    """Symmetric-lower -> general pattern map: ``general.values = lower.values[src]``."""

    general: CsMatrix
    src: np.ndarray


def expand_pattern(A: CsMatrix) -> Expansion:
    """The pattern half of ``to_general`` (sparsecore.py:263-273), with the value map.

    Pure reindexing (values move bitwise), so the device can rebuild the general values
    of every later system from its lower-triangle values with one gather.
    """
    if A.symmetry == GENERAL:
        return Expansion(A, np.arange(A.nnz, dtype=np.int64))
    rows = A.row_of_entry()
    strict = np.flatnonzero(rows != A.col_idx)
    r = np.concatenate([rows, A.col_idx[strict]])
    c = np.concatenate([A.col_idx, rows[strict]])
    src = np.concatenate([np.arange(A.nnz, dtype=np.int64), strict])
    key = np.lexsort((c, r))
    r, c, src = r[key], c[key], src[key]
    row_ptr = np.zeros(A.n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=A.n_rows), out=row_ptr[1:])
    G = CsMatrix(A.n_rows, A.n_cols, row_ptr, c, A.values[src], GENERAL, _checked=True)
    return Expansion(G, src)


def to_general(A: CsMatrix) -> CsMatrix:
    """Explicit general storage of a symmetric-lower matrix (sparsecore.py:263)."""
    if A.symmetry == GENERAL:
        return A
    return expand_pattern(A).general


def lower_map(G: CsMatrix):
    """Symmetric-lower storage of a structurally symmetric general pattern.

    Returns ``(row_ptr, col_idx, gen_src)`` with ``G.values == lower_values[gen_src]`` for a
    numerically symmetric matrix (the inverse of :func:`expand_pattern`), or None when the
    pattern is not structurally symmetric.
    """
    n = G.n_rows
    if G.n_cols != n:
        return None
    rows = G.row_of_entry()
    cols = G.col_idx
    low = cols <= rows
    lidx = np.cumsum(low) - 1
    lrows, lcols = rows[low], cols[low]
    l_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(lrows, minlength=n), out=l_ptr[1:])
    key_low = lrows * n + lcols          # ascending (row-major)
    up = ~low
    key_up = cols[up] * n + rows[up]     # mirrored position
    pos = np.searchsorted(key_low, key_up)
    if pos.size and (np.any(pos >= key_low.size) or np.any(key_low[np.minimum(pos, key_low.size - 1)] != key_up)):
        return None
    # every strict-lower entry must have its mirror too
    if int(np.count_nonzero(up)) != int(np.count_nonzero(lrows != lcols)):
        return None
    gen_src = np.empty(G.nnz, dtype=np.int64)
    gen_src[low] = lidx[low]
    gen_src[up] = pos
    return l_ptr, lcols.astype(np.int64), gen_src
