"""GPU: the straggler hand-off of batched FGMRES (krylov.cu, resume_handed).

Once at most T systems of a lockstep batch still iterate, they leave the batch mid-cycle with
their whole Krylov state and finish on single-system helper handles (concurrent streams).
Here T = 4 on a 20-system batch of the BASELINE-size reference goldens: every system against
the REFERENCE's own results (trigger, iterations +-1, rr bar, converged), and against the same
batch run fully in lockstep (iterations +-1, untriggered x bitwise).  The benchmarked B = 64
batch with the default T is checked against the oracle in test_gpu_scale.py.
"""

import numpy as np
import pytest

from large_golden import M, available, check_report, load, rr_floor, sequence

pytestmark = pytest.mark.gpu

@pytest.mark.parametrize("case", [c for c in ("activsg2000p", "activsg200p") if available(c)])
def test_handoff_against_reference(case, monkeypatch):
    """Up to 4 stragglers of a 20-system batch finish on concurrent helpers; every system
    stays within the reference bars, and forcing the lockstep batch gives the same iteration
    counts within +-1."""
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200 import factorize, to_general
    from paper_2401_13926_b200.device import DeviceSystem
    monkeypatch.setenv("KKT_HANDOFF", "4")
    g = load(case)
    seq = sequence(case)
    f, _ = factorize(to_general(seq.matrix(0)))
    dev = DeviceSystem(f, batch=M)
    vals = np.stack([seq.values(k) for k in range(M)])
    rhs = np.stack([seq.rhs(k) for k in range(M)])
    deltas = [1e-10] * M
    x = np.empty_like(rhs)
    reps = dev.step(vals, nat.LAYOUT_SYMMETRIC_LOWER, rhs, x, False, 10, 10, deltas, stats=True)
    x2 = np.empty_like(rhs)
    reps2 = dev.step(vals, nat.LAYOUT_SYMMETRIC_LOWER, rhs, x2, False, 10, 10, deltas, stats=True,
                     handoff=False)
    assert sum(r.handed_off for r in reps) >= 2
    assert sum(r.handed_off for r in reps2) == 0
    for k, (rep, rep2) in enumerate(zip(reps, reps2)):
        err2, r2 = rep.stats_after[0], rep.stats_after[4]
        rr = err2 / r2 if rep.triggered else rep.stats_before[0] / rep.stats_before[4]
        K = seq.matrix(k)
        fl = rr_floor(K.row_ptr, K.col_idx, K.values, x[k], rhs[k])
        check_report(dict(triggered=rep.triggered, iterations=rep.iterations, rr=rr,
                          converged=rep.converged, floor=fl), g["refine_1e-10"][k], (case, k), 1e-10)
        assert abs(rep.iterations - rep2.iterations) <= 1, k
        if not rep.triggered:
            assert np.array_equal(x[k], x2[k])
    dev.close()
