"""Host analysis (C++, kkt_analyze) is bit-exact with the reference's factorize.

Pinned against tests/golden/*.npz, which tests/golden/make_golden.py produced by running the
reference kktsolve.direct_lu.factorize (direct_lu.py:116-294)."""

import numpy as np
import pytest

from conftest import FACTOR_KEYS, factor_dict, golden, lower_matrix
from paper_2401_13926_b200 import (SingularMatrixError, Triplets, factorize, from_dense,
                                   from_triplets, identity, to_general)


@pytest.mark.parametrize("case", ["standard_trace", "acopf_tiny", "acopf_small"])
def test_sequence_analysis_bitwise(case):
    g = golden(case)
    f, d = factorize(to_general(lower_matrix(g, 0)))
    got = factor_dict(f)
    for k in FACTOR_KEYS:
        assert np.array_equal(got[k], g[f"f0_{k}"]), k
    assert np.array_equal([d.max_abs_pivot, d.min_abs_pivot, d.zero_pivots_patched,
                           d.growth_estimate], g["f0_diag"])


def test_symmetric_lower_input_is_expanded():
    g = golden("standard_trace")
    f, _ = factorize(lower_matrix(g, 0))  # factorize expands sym-lower itself (:132)
    assert np.array_equal(f._Li, g["f0_Li"]) and np.array_equal(f._Lx, g["f0_Lx"])


def test_random_sparse_bitwise():
    g = golden("random_sparse")
    from paper_2401_13926_b200.sparse import CsMatrix
    for s in range(int(g["count"][0])):
        rp = g[f"r{s}_row_ptr"]
        n = rp.size - 1
        A = CsMatrix(n, n, rp, g[f"r{s}_col_idx"], g[f"r{s}_values"])
        f, d = factorize(A)
        got = factor_dict(f)
        for k in FACTOR_KEYS:
            assert np.array_equal(got[k], g[f"r{s}_{k}"]), (s, k)
        assert np.array_equal([d.max_abs_pivot, d.min_abs_pivot, d.zero_pivots_patched,
                               d.growth_estimate], g[f"r{s}_diag"])


def test_identity_and_forced_swap():
    f, d = factorize(identity(3))
    assert np.array_equal(f.L.to_dense(), np.eye(3))
    assert np.array_equal(f.U.to_dense(), np.eye(3))
    assert d.zero_pivots_patched == 0
    g = golden("edge_cases")
    s, _ = factorize(from_dense(np.array([[0.0, 1.0], [1.0, 0.0]])))
    assert np.array_equal(s.row_perm.perm, g["swap_row_perm"])
    assert np.array_equal(s.col_perm.perm, g["swap_col_perm"])
    assert np.array_equal(s.L.to_dense(), np.eye(2)) and np.array_equal(s.U.to_dense(), np.eye(2))


def test_singular_errors():
    with pytest.raises(SingularMatrixError):
        factorize(from_triplets(Triplets.from_entries(2, 2, [(0, 0, 1.0)])))
    with pytest.raises(SingularMatrixError):
        factorize(from_dense(np.array([[1.0, 2.0], [2.0, 4.0]])))
    with pytest.raises(ValueError):
        factorize(identity(3), pivot_tol=0.0)


def test_schedule_stats_reported():
    g = golden("acopf_small")
    f, _ = factorize(lower_matrix(g, 0))
    st = f.stats
    assert st["nnz_L"] == g["f0_Li"].size and st["refactor_levels"] >= 1
    assert st["update_pairs"] == int(sum(np.diff(g["f0_Lp"])[g["f0_so_data"]]))
