"""The CPU oracle is pinned to the reference's own outputs (tests/golden, made by running
kktsolve itself).  Bitwise for refactorize / lu_solve / spmv; FGMRES-IR iteration counts
within +-1 (the oracle's dot products are sequential, the reference's are BLAS)."""

import numpy as np
import pytest

from conftest import FACTOR_KEYS, golden
from oracle import oracle
from paper_2401_13926_b200.sparse import SYMMETRIC_LOWER, CsMatrix, expand_pattern


def _factors(g):
    arrays = {k: g[f"f0_{k}"] for k in FACTOR_KEYS}
    n = int(g["n"][0])
    K = CsMatrix(n, n, g["K_row_ptr"], g["K_col_idx"], g["K_values"][0], SYMMETRIC_LOWER)
    ex = expand_pattern(K)
    return oracle.OracleFactors(arrays, ex.general.row_ptr), ex


@pytest.mark.parametrize("case", ["standard_trace", "acopf_tiny", "acopf_small"])
def test_oracle_refactor_solve_spmv_bitwise(case):
    g = golden(case)
    of, ex = _factors(g)
    for i in range(g["K_values"].shape[0]):
        kv = g["K_values"][i]
        d = of.refactorize(kv[ex.src])
        assert np.array_equal(d, g["refactor_diag"][i]), i
        if f"s{i}_Lx" in g:
            assert np.array_equal(of.a["Lx"], g[f"s{i}_Lx"])
            assert np.array_equal(of.a["Ux"], g[f"s{i}_Ux"])
            assert np.array_equal(of.a["Udiag"], g[f"s{i}_Udiag"])
        assert np.array_equal(of.lu_solve(g["rhs"][i]), g["x0"][i]), i
        y = oracle.spmv(g["K_row_ptr"], g["K_col_idx"], kv, g["x0"][i])
        assert np.array_equal(y, g["spmv_K_x0"][i]), i


@pytest.mark.parametrize("case", ["standard_trace", "acopf_tiny", "acopf_small"])
def test_oracle_refine_matches_reference(case):
    g = golden(case)
    of, ex = _factors(g)
    for tag, delta in (("1e-10", 1e-10), ("1e-14", 1e-14)):
        ref = g[f"refine_{tag}_report"]
        for i in range(g["K_values"].shape[0]):
            kv = g["K_values"][i]
            of.refactorize(kv[ex.src])
            x0 = of.lu_solve(g["rhs"][i])
            x, rep = of.refine_fgmres(g["K_row_ptr"], g["K_col_idx"], kv, g["rhs"][i], x0, delta)
            assert rep["triggered"] == bool(ref[i, 0]), (tag, i)
            assert abs(rep["iterations"] - int(ref[i, 1])) <= 1, (tag, i)
            if rep["triggered"]:
                xr = g[f"refine_{tag}_x"][i]
                assert np.linalg.norm(x - xr) <= 1e-6 * np.linalg.norm(xr) + 1e-12


def test_oracle_inf_norm():
    g = golden("standard_trace")
    v = oracle.inf_norm(g["K_row_ptr"], g["K_col_idx"], g["K_values"][0])
    n = int(g["n"][0])
    K = CsMatrix(n, n, g["K_row_ptr"], g["K_col_idx"], g["K_values"][0], SYMMETRIC_LOWER)
    assert abs(v - np.abs(K.to_dense()).sum(axis=1).max()) <= 1e-12 * v
