"""GPU: the sm_100a path against the REFERENCE at BASELINE sizes (tests/golden/large_*.npz).

For every system k = 0..19 of configs[0] (N = 9,030), configs[1] (N = 90,320) and the
pivoting variants (row_perm != col_perm; direct_lu.py:209-223):

* refactorize on the device: _Lx / _Ux / _Udiag BITWISE the reference's (SHA-256), and the
  LuDiagnostics exactly;
* lu_solve: x0 BITWISE the reference's (SHA-256);
* refine_fgmres (kkt_dev_step, one device-controlled graph) at delta = 1e-10 and at the
  barrier-tied delta(mu_k): trigger equal, FGMRES iterations within +-1, true residual
  rr <= max(1.5 rr_ref, 4 eps, 1e-3 delta), converged equal;
* the same 20 systems as ONE batched handle (nb = 20): every system's factors and x0 bitwise
  the reference's, the batched refine within the same bars.
"""

import numpy as np
import pytest

from large_golden import (CASES, M, available, barrier_delta, check_report, load, rr_floor,
                          sequence, sha)
from paper_2401_13926_b200 import _native as nat
from paper_2401_13926_b200 import factorize, to_general

pytestmark = pytest.mark.gpu
CASE_IDS = [c for c in CASES if available(c)]
LOWER = nat.LAYOUT_SYMMETRIC_LOWER


def _rr(stats_after):
    err2, r2 = stats_after[0], stats_after[4]
    return err2 / r2 if r2 > 0 else 0.0


@pytest.mark.parametrize("case", CASE_IDS)
def test_single_system_sequence(case):
    g = load(case)
    seq = sequence(case)
    f, _ = factorize(to_general(seq.matrix(0)))
    dev = f.device()
    torch = dev.torch
    for k in range(M):
        vals = np.ascontiguousarray(seq.values(k))
        r = seq.rhs(k)
        # refactorize -> factors bitwise
        K = seq.matrix(k)
        d = dev.refactor_matrix(K)
        assert np.array_equal([d.max_abs_pivot, d.min_abs_pivot, d.zero_pivots_patched,
                               d.growth_estimate], g["refactor_diag"][k]), k
        Lx, Ux, Ud = dev.download_factors()
        assert [sha(Lx), sha(Ux), sha(Ud)] == list(g["sha_factors"][k]), k
        x0 = dev.solve_host(r)
        assert sha(x0) == str(g["sha_x0"][k]), k
        # the whole per-system step (refactor -> solve -> refine) in one call per tolerance
        for tag, delta in (("1e-10", 1e-10), ("barrier", barrier_delta(seq, k))):
            x = np.empty_like(r)
            rep = dev.step(vals, LOWER, r, x, False, 10, 10, delta, stats=True)
            rr = _rr(rep.stats_after) if rep.triggered else _rr(rep.stats_before)
            fl = rr_floor(K.row_ptr, K.col_idx, K.values, x, r)
            check_report(dict(triggered=rep.triggered, iterations=rep.iterations, rr=rr,
                              converged=rep.converged, floor=fl), g[f"refine_{tag}"][k],
                         (case, k, tag), delta)
            if f"s{k}_x_{tag}" in g and not rep.triggered:
                assert np.array_equal(x, g[f"s{k}_x_{tag}"])
    del torch


@pytest.mark.parametrize("case", CASE_IDS)
def test_batched_sequence(case):
    from paper_2401_13926_b200.device import DeviceSystem
    g = load(case)
    seq = sequence(case)
    f, _ = factorize(to_general(seq.matrix(0)))
    dev = DeviceSystem(f, batch=M)
    torch = dev.torch
    vals = np.stack([seq.values(k) for k in range(M)])
    rhs = np.stack([seq.rhs(k) for k in range(M)])
    with torch.cuda.stream(dev.stream):
        v_t = torch.from_numpy(vals).to(dev.device)
        r_t = torch.from_numpy(rhs).to(dev.device)
        x0_t = torch.empty_like(r_t)
    diag = dev.refactor_batch(v_t, LOWER)
    assert np.array_equal(diag, g["refactor_diag"])
    Lx, Ux, Ud = dev.download_factors_batch()
    for k in range(M):
        assert [sha(Lx[k]), sha(Ux[k]), sha(Ud[k])] == list(g["sha_factors"][k]), k
    dev.solve_device(r_t, x0_t)
    x0 = dev.d2h(x0_t)
    for k in range(M):
        assert sha(x0[k]) == str(g["sha_x0"][k]), k
    for tag in ("1e-10", "barrier"):
        deltas = [1e-10 if tag == "1e-10" else barrier_delta(seq, k) for k in range(M)]
        x = np.empty_like(rhs)
        reps = dev.step(vals, LOWER, rhs, x, False, 10, 10, deltas, stats=True)
        for k, rep in enumerate(reps):
            rr = _rr(rep.stats_after) if rep.triggered else _rr(rep.stats_before)
            K = seq.matrix(k)
            fl = rr_floor(K.row_ptr, K.col_idx, K.values, x[k], rhs[k])
            check_report(dict(triggered=rep.triggered, iterations=rep.iterations, rr=rr,
                              converged=rep.converged, floor=fl), g[f"refine_{tag}"][k],
                         (case, k, tag), deltas[k])
    dev.close()
