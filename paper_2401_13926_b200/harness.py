"""The per-system loop of ``harness._run_direct_family`` (harness.py:217-269) on the B200.

``run_refactor_ir`` walks a same-pattern sequence exactly like the reference's
``refactor_ir_fgmres`` strategy — analyze system 0 on the host, then per system:
refactorize -> lu_solve -> refine_fgmres — and returns the reference's row metrics.
Two execution modes:

* ``mode="dropin"``  : through this package's reference-compatible functions (numpy in/out);
* ``mode="device"``  : one ``kkt_dev_step`` C call per system (values + rhs uploaded,
  x downloaded), the fast path the benchmark's ``e2e`` leg measures.

Row metrics (nsr / nrbe / rr) are computed by the same device residual pass for both modes.
The optional ``tolerance`` policy maps each system's mu to delta_tol (barrier-tied IR).
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .direct_lu import factorize, lu_solve, refactorize
from .refine import (FixedTolerance, RefinementConfig, config_for_mu, refine_fgmres,
                     refine_richardson)
from .sparse import SYMMETRIC_LOWER, CsMatrix, to_general


class SequenceError(ValueError):
    """Invalid sequence manifest or pattern drift (harness.py SequenceError)."""


@dataclass
class SequenceItem:
    K: CsMatrix
    rhs: np.ndarray
    matrix_path: str | None = None
    rhs_path: str | None = None


@dataclass
class MatrixSequence:
    name: str
    items: list
    metadata: dict = field(default_factory=dict)


def _lower_nnz(K: CsMatrix) -> int:
    if K.symmetry == SYMMETRIC_LOWER:
        return K.nnz
    rows = np.repeat(np.arange(K.n_rows), np.diff(K.row_ptr))
    return int(np.count_nonzero(rows >= K.col_idx))


def load_sequence(manifest_path: str) -> MatrixSequence:
    """A manifest's systems through the C++ Matrix Market reader, validating the shared
    pattern (harness.load_sequence, harness.py:118-146)."""
    from .mmio import load_matrix_market, load_vector
    with open(manifest_path, "r") as fh:
        manifest = json.load(fh)
    systems = manifest.get("systems", [])
    if not systems:
        raise SequenceError("sequence must contain at least one system")
    base = os.path.dirname(os.path.abspath(manifest_path))
    items: list[SequenceItem] = []
    for i, entry in enumerate(systems):
        mpath = os.path.join(base, entry["matrix"])
        rpath = os.path.join(base, entry["rhs"])
        K = load_matrix_market(mpath)
        rhs = load_vector(rpath)
        if rhs.size != K.n_rows:
            raise SequenceError(f"system {i}: rhs length {rhs.size} does not "
                                f"match matrix dimension {K.n_rows}")
        if items and not K.same_pattern(items[0].K):
            raise SequenceError(f"system {i}: sparsity pattern differs from system 0")
        items.append(SequenceItem(K=K, rhs=rhs, matrix_path=mpath, rhs_path=rpath))
    metadata = {"N": items[0].K.n_rows, "nnz": _lower_nnz(items[0].K)}
    for key in ("n", "m", "mu"):
        if key in manifest:
            metadata[key] = manifest[key]
    return MatrixSequence(name=manifest.get("name", "sequence"), items=items, metadata=metadata)


@dataclass
class RowMetrics:
    """harness.RowMetrics (harness.py:85-97)."""

    index: int
    nsr_before: float
    nsr_after: float
    nrbe: float
    rr: float
    ir_iterations: int
    triangular_solves: int
    factorize_time_s: float
    solve_time_s: float
    refine_time_s: float
    converged: bool


def run_refactor_ir(matrices, rhss, cfg: RefinementConfig | None = None, mus=None,
                    tolerance=None, mode: str = "device", refresh_after: int = 1,
                    method: str = "fgmres"):
    """Run the refactor_ir_fgmres (``method="fgmres"``) or refactor_ir_richardson
    (``"richardson"``, refine.py:135; drop-in mode) strategy; returns (rows, factors)."""
    cfg = cfg or RefinementConfig()
    if method not in ("fgmres", "richardson"):
        raise ValueError(f"unknown refinement method {method!r}")
    refine = refine_fgmres if method == "fgmres" else refine_richardson
    if method == "richardson":
        mode = "dropin"
    policy = tolerance or FixedTolerance(cfg.delta_tol)
    rows: list[RowMetrics] = []
    factors = None
    dev = None
    for idx, (K, r) in enumerate(zip(matrices, rhss)):
        r = np.asarray(r, dtype=np.float64)
        mu = None if mus is None else mus[idx]
        rc = config_for_mu(cfg, policy, mu)
        if factors is None or idx < refresh_after:
            t0 = time.perf_counter()
            factors, _ = factorize(to_general(K))
            dev = factors.device(restart_m=rc.krylov.m)
            t_fact = time.perf_counter() - t0
            count0 = factors.triangular_solve_count
            t0 = time.perf_counter()
            x0 = lu_solve(factors, r)
            t_solve = time.perf_counter() - t0
            t0 = time.perf_counter()
            x, rep = refine(K, factors, x0, r, rc)
            t_ref = time.perf_counter() - t0
            iters, conv = rep.ir_iterations, rep.converged
            nsr_b, nsr_a = rep.nsr_before, rep.nsr_after
            tsolves = factors.triangular_solve_count - count0
        elif mode == "dropin":
            t0 = time.perf_counter()
            refactorize(factors, to_general(K))
            t_fact = time.perf_counter() - t0
            count0 = factors.triangular_solve_count
            t0 = time.perf_counter()
            x0 = lu_solve(factors, r)
            t_solve = time.perf_counter() - t0
            t0 = time.perf_counter()
            x, rep = refine(K, factors, x0, r, rc)
            t_ref = time.perf_counter() - t0
            iters, conv = rep.ir_iterations, rep.converged
            nsr_b, nsr_a = rep.nsr_before, rep.nsr_after
            tsolves = factors.triangular_solve_count - count0
        else:
            layout = nat.LAYOUT_SYMMETRIC_LOWER if K.symmetry == SYMMETRIC_LOWER \
                else nat.LAYOUT_GENERAL
            if layout == nat.LAYOUT_SYMMETRIC_LOWER:
                dev._layout_of(K)
            x = np.empty_like(r)
            t0 = time.perf_counter()
            krep = dev.step(np.ascontiguousarray(K.values), layout, r, x, False,
                            rc.krylov.m, rc.krylov.max_outer, rc.delta_tol)
            t_fact, t_solve, t_ref = time.perf_counter() - t0, 0.0, 0.0
            factors._host_vals = None
            factors.from_refactorization = True
            iters = krep.iterations
            conv = bool(krep.converged)
            tsolves = 1 + iters
            factors.triangular_solve_count += tsolves
            nsr_b = nsr_a = float("nan")
        # quality metrics of the returned x, one device residual pass (harness.py:249-266)
        dev.set_operator(K)
        dev.h2d(dev.r, r)
        dev.h2d(dev.x, x)
        s = dev.residual_stats_device(dev.r, dev.x)
        if np.isnan(nsr_a):
            nsr_a = s.nsr()
            nsr_b = nsr_a if iters == 0 else float("nan")
        if not np.all(np.isfinite(x)):
            conv = False
        rr = s.err2 / s.r2 if s.r2 > 0 else 0.0
        rows.append(RowMetrics(idx, nsr_b, nsr_a, s.nrbe(), rr, iters, tsolves, t_fact,
                               t_solve, t_ref, conv))
    return rows, factors
