"""CPU: the host analysis and the oracle against the REFERENCE at BASELINE sizes.

configs[0] (ACTIVSg200, N = 9,030) and configs[1] (ACTIVSg2000, N = 90,320) of the
ACOPF-shaped family, plus pivoting variants where the reference's threshold pivoting picks
off-diagonal pivots (activsg200p: 1,411; activsg2000q: ~3,200; activsg2000p: 7,610) — the
``row_perm != col_perm`` regime of direct_lu.py:209-223.  Goldens: tests/golden/large_*.npz
made by tests/golden/make_golden_large.py from the reference package itself.

* ``kkt_analyze`` (C++) == ``factorize`` (direct_lu.py:116-294): every LuFactors array
  bitwise (full arrays at 9k, SHA-256 at 90k) and the LuDiagnostics.
* the oracle (oracle/kkt_oracle.c): refactorize factors bitwise (SHA-256 of _Lx/_Ux/_Udiag),
  lu_solve bitwise, refine_fgmres trigger / iterations / residual vs the reference's reports.
"""

import numpy as np
import pytest

from conftest import FACTOR_KEYS, factor_dict
from large_golden import CASES, M, available, barrier_delta, check_report, load, sequence, sha
from paper_2401_13926_b200 import factorize, to_general

CASE_IDS = [c for c in CASES if available(c)]


@pytest.mark.parametrize("case", CASE_IDS)
def test_analysis_matches_reference(case):
    g = load(case)
    seq = sequence(case)
    f, d = factorize(to_general(seq.matrix(0)))
    got = factor_dict(f)
    for k in FACTOR_KEYS:
        if f"f0_{k}" in g:
            assert np.array_equal(got[k], g[f"f0_{k}"]), k
        assert sha(got[k]) == str(g[f"sha_{k}"]), k
    assert np.array_equal([d.max_abs_pivot, d.min_abs_pivot, d.zero_pivots_patched,
                           d.growth_estimate], g["f0_diag"])
    assert int(np.sum(f.row_perm.perm != f.col_perm.perm)) == int(g["offdiag_pivots"][0])


@pytest.mark.parametrize("case", CASE_IDS)
def test_oracle_matches_reference(case):
    from oracle import oracle
    from paper_2401_13926_b200.sparse import expand_pattern
    g = load(case)
    seq = sequence(case)
    K0 = seq.matrix(0)
    f, _ = factorize(to_general(K0))
    ex = expand_pattern(K0)
    of = oracle.OracleFactors(factor_dict(f), ex.general.row_ptr)
    # the 1.9 G-pair case checks a subset of the systems to keep the CPU suite short
    ks = range(M) if f.stats["update_pairs"] < 2e8 else (0, 10, 19)
    for k in ks:
        K = seq.matrix(k)
        r = seq.rhs(k)
        d = of.refactorize(K.values[ex.src])
        assert np.array_equal(d, g["refactor_diag"][k]), k
        assert [sha(of.a["Lx"]), sha(of.a["Ux"]), sha(of.a["Udiag"])] == list(g["sha_factors"][k]), k
        x0 = of.lu_solve(r)
        assert sha(x0) == str(g["sha_x0"][k]), k
        for tag, delta in (("1e-10", 1e-10), ("barrier", barrier_delta(seq, k))):
            x, rep = of.refine_fgmres(K.row_ptr, K.col_idx, K.values, r, x0, delta)
            rr = np.linalg.norm(r - oracle.spmv(K.row_ptr, K.col_idx, K.values, x)) / np.linalg.norm(r)
            check_report(dict(triggered=rep["triggered"], iterations=rep["iterations"], rr=rr,
                              converged=rep["converged"]), g[f"refine_{tag}"][k], (case, k, tag), delta)
