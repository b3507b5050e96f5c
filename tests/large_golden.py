"""Helpers for the BASELINE-size reference goldens (tests/golden/large_<case>.npz).

The fixtures are outputs of the REFERENCE itself (tests/golden/make_golden_large.py imports
kktsolve from /root/reference in the build container); the inputs are rebuilt here from the
deterministic generator (acopf.make_sequence), so only the reference's outputs are stored.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from conftest import GOLDEN

CASES = {  # case -> (acopf config, imbalance_frac)
    "activsg200": ("activsg200", 1.0),
    "activsg200p": ("activsg200", 0.5),
    "activsg2000": ("activsg2000", 1.0),
    "activsg2000q": ("activsg2000", 0.9),
    "activsg2000p": ("activsg2000", 0.75),
}
M = 20
REPORT = ["triggered", "ir_iterations", "triangular_solves_used", "nsr_before", "nsr_after",
          "rr_final", "nrbe_final", "converged", "rr_true"]


def available(case: str) -> bool:
    return os.path.exists(os.path.join(GOLDEN, f"large_{case}.npz"))


def load(case: str):
    return np.load(os.path.join(GOLDEN, f"large_{case}.npz"))


def meta(case: str) -> dict:
    return json.load(open(os.path.join(GOLDEN, f"large_{case}.json")))


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    a = a.astype(np.float64 if a.dtype.kind == "f" else np.int64, copy=False)
    return hashlib.sha256(a.tobytes()).hexdigest()


_SEQ = {}


def sequence(case: str):
    if case not in _SEQ:
        from paper_2401_13926_b200.acopf import make_sequence
        cfg, frac = CASES[case]
        _SEQ.clear()
        _SEQ[case] = make_sequence(cfg, seed=0, length=M, imbalance_frac=frac)
    return _SEQ[case]


def barrier_delta(seq, k: int) -> float:
    from paper_2401_13926_b200.refine import BarrierTiedTolerance
    return BarrierTiedTolerance()(seq.mu(k))


# The reference's own final residual is reproducible only to a factor RR_SPREAD under another
# summation order: the plain-C oracle (same algorithm, sequential dots instead of OpenBLAS)
# lands at up to 2.06x the reference's rr on these goldens at EQUAL iteration counts
# (activsg200p k = 18: 1.87e-14 vs 3.85e-14; profiles/r2_rr_spread.txt, tools/rr_spread.py).
RR_SPREAD = 2.5


def rr_floor(K_rp, K_ci, K_vals, x, r) -> float:
    """The rounding floor of the residual evaluation itself: eps * || |K| |x| ||_2 / ||r||_2.
    Computing r - K x in double carries an error of that size, so two residuals below it differ
    only by rounding noise (ACTIVSg10k k = 18: the oracle's rr is 1.96e-13 with a floor of
    1.1e-12)."""
    from oracle import oracle
    ax = oracle.spmv(K_rp, K_ci, np.abs(K_vals), np.abs(x))
    nr = np.linalg.norm(r)
    return float(np.finfo(float).eps * np.linalg.norm(ax) / nr) if nr > 0 else 0.0


def rr_bound(rr_ref: float, delta: float, same_iterations: bool = True, floor: float = 0.0) -> float:
    """The residual parity bar.

    Equal iteration counts: rr <= max(RR_SPREAD rr_ref, 4 eps, floor) — the measured
    reproducibility of the reference's rr under reassociated reductions (SURVEY.md §7 hard
    part 5), and the rounding floor of evaluating r - K x (`rr_floor`), below which residuals
    carry no information.
    One iteration fewer than the reference (the +-1 allowance): that iteration's gain is not
    made, so rr is bounded by the stopping rule instead — rr <= delta (the oracle itself stops
    one iteration early on activsg2000p barrier k = 17 and lands at 89x the reference's rr,
    5.98e-11 for delta = 2e-9).
    """
    eps = np.finfo(float).eps
    if not same_iterations:
        return max(RR_SPREAD * rr_ref, delta, floor)
    return max(RR_SPREAD * rr_ref, 4 * eps, floor)


def check_report(got: dict, ref_row, tag: str, delta: float):
    """trigger equal, iterations within +-1, rr <= rr_bound, converged equal."""
    r = dict(zip(REPORT, ref_row))
    assert bool(got["triggered"]) == bool(r["triggered"]), (tag, got, r)
    assert abs(got["iterations"] - r["ir_iterations"]) <= 1, (tag, got, r)
    same = got["iterations"] >= r["ir_iterations"]
    assert got["rr"] <= rr_bound(r["rr_true"], delta, same, got.get("floor", 0.0)), (tag, got, r)
    assert bool(got["converged"]) == bool(r["converged"]), (tag, got, r)
