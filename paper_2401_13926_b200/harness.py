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
from .device import ResidualStats
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
    """Entries on or below the diagonal (the symmetric-lower storage size)."""
    if K.symmetry == SYMMETRIC_LOWER:
        return K.nnz
    row_of = np.repeat(np.arange(K.n_rows, dtype=np.int64), np.diff(K.row_ptr))
    return int((K.col_idx <= row_of).sum())


def load_sequence(manifest_path: str, workers: int | None = None) -> MatrixSequence:
    """Load a manifest's systems (harness.load_sequence, harness.py:118-146).

    The Matrix Market files are parsed concurrently by the C++ reader (``kkt_mm_*`` releases
    the GIL), then validated in manifest order so the first failing system raises the
    reference's ``SequenceError`` (rhs length before pattern).  Every system after the first
    shares system 0's pattern arrays: a sequence costs one pattern plus M value arrays.
    """
    from concurrent.futures import ThreadPoolExecutor

    from .mmio import load_matrix_market, load_vector
    with open(manifest_path, "r") as fh:
        manifest = json.load(fh)
    entries = manifest.get("systems", [])
    if not entries:
        raise SequenceError("sequence must contain at least one system")
    base = os.path.dirname(os.path.abspath(manifest_path))
    paths = [(os.path.join(base, e["matrix"]), os.path.join(base, e["rhs"])) for e in entries]

    def parse(pair):
        try:
            return load_matrix_market(pair[0]), load_vector(pair[1]), None
        except Exception as exc:  # raised in manifest order below
            return None, None, exc

    with ThreadPoolExecutor(max_workers=workers or min(8, len(paths))) as ex:
        parsed = list(ex.map(parse, paths))
    items: list[SequenceItem] = []
    K0 = None
    for i, ((mpath, rpath), (K, rhs, err)) in enumerate(zip(paths, parsed)):
        if err is not None:
            raise err
        if rhs.size != K.n_rows:
            raise SequenceError(f"system {i}: rhs length {rhs.size} does not "
                                f"match matrix dimension {K.n_rows}")
        if K0 is None:
            K0 = K
        elif not K.same_pattern(K0):
            raise SequenceError(f"system {i}: sparsity pattern differs from system 0")
        else:
            K = K0.with_values(K.values)
        items.append(SequenceItem(K=K, rhs=rhs, matrix_path=mpath, rhs_path=rpath))
    metadata = {"N": K0.n_rows, "nnz": _lower_nnz(K0)}
    metadata.update({k: manifest[k] for k in ("n", "m", "mu") if k in manifest})
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
                            rc.krylov.m, rc.krylov.max_outer, rc.delta_tol, stats=True)
            t_fact, t_solve, t_ref = time.perf_counter() - t0, 0.0, 0.0
            factors._host_vals = None
            factors.from_refactorization = True
            iters = krep.iterations
            conv = bool(krep.converged)
            tsolves = 1 + iters
            factors.triangular_solve_count += tsolves
            nsr_b = ResidualStats(*krep.stats_before).nsr()
            nsr_a = ResidualStats(*krep.stats_after).nsr() if krep.triggered else nsr_b
        # quality metrics of the returned x, one device residual pass (harness.py:249-266)
        dev.set_operator(K)
        dev.h2d(dev.r, r)
        dev.h2d(dev.x, x)
        s = dev.residual_stats_device(dev.r, dev.x)
        if not np.all(np.isfinite(x)):
            conv = False
        rr = s.err2 / s.r2 if s.r2 > 0 else 0.0
        rows.append(RowMetrics(idx, nsr_b, nsr_a, s.nrbe(), rr, iters, tsolves, t_fact,
                               t_solve, t_ref, conv))
    return rows, factors
