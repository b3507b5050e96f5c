"""Richardson iterative refinement on the device (refine.refine_richardson, refine.py:135-205;
SURVEY.md §8f row 2) against the reference's own outputs (tests/golden, make_golden.py).

Every iterate is lu_solve (bitwise) + an elementwise add (bitwise) + the reference-order
residual, so when the stopping decisions agree the returned x is bitwise the reference's;
the decisions use tree-reduced 2-norms, so the report's norm ratios are compared to 1e-12.
"""

import numpy as np
import pytest

from conftest import golden, lower_matrix
from paper_2401_13926_b200 import (RefinementConfig, factorize, lu_solve, refactorize,
                                   refine_richardson, to_general)

pytestmark = pytest.mark.gpu

CFGS = {"1e-10": dict(delta_tol=1e-10), "1e-14": dict(delta_tol=1e-14),
        "nsr": dict(delta_tol=1e-10, richardson_stop="nsr_ratio")}


@pytest.mark.parametrize("case", ["standard_trace", "acopf_tiny", "acopf_small"])
@pytest.mark.parametrize("tag", list(CFGS))
def test_refine_richardson_matches_reference(case, tag):
    g = golden(case)
    ref = g[f"richardson_{tag}_report"]
    xref = g[f"richardson_{tag}_x"]
    f, _ = factorize(to_general(lower_matrix(g, 0)))
    cfg = RefinementConfig(**CFGS[tag])
    for i in range(g["K_values"].shape[0]):
        K = lower_matrix(g, i)
        r = g["rhs"][i]
        refactorize(f, to_general(K))
        x0 = lu_solve(f, r)
        c0 = f.triangular_solve_count
        x, rep = refine_richardson(K, f, x0, r, cfg)
        assert rep.triggered == bool(ref[i, 0]), i
        assert rep.ir_iterations == int(ref[i, 1]), (i, rep.ir_iterations, ref[i, 1])
        assert rep.triangular_solves_used == int(ref[i, 2]) == f.triangular_solve_count - c0
        assert rep.converged == bool(ref[i, 7]) and rep.diverged == bool(ref[i, 8]), i
        assert np.array_equal(x, xref[i]), i
        if rep.triggered:
            assert rep.nsr_before == pytest.approx(ref[i, 3], rel=1e-12)
            assert rep.nsr_after == pytest.approx(ref[i, 4], rel=1e-12, abs=1e-300)
            assert rep.rr_final == pytest.approx(ref[i, 5], rel=1e-10, abs=1e-300)
            assert rep.nrbe_final == pytest.approx(ref[i, 6], rel=1e-10, abs=1e-300)


def test_harness_richardson_rows():
    """The refactor_ir_richardson strategy through the harness: per-row iterations and
    triangular-solve counts equal the reference's (harness.py:217-269 with refine_richardson)."""
    from paper_2401_13926_b200.harness import run_refactor_ir
    g = golden("acopf_small")
    M = g["K_values"].shape[0]
    Ks = [lower_matrix(g, i) for i in range(M)]
    rows, _ = run_refactor_ir(Ks, list(g["rhs"]), RefinementConfig(delta_tol=1e-10),
                              method="richardson")
    ref = g["richardson_1e-10_report"]
    for i in range(1, M):
        assert rows[i].ir_iterations == int(ref[i, 1]), i
        assert rows[i].triangular_solves == 1 + int(ref[i, 2]), i
