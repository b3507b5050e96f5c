"""GPU: parity where the headline numbers come from (bench.py's exact workloads).

* The bench batch: B = 64 ACTIVSg10k-shaped systems (N = 238,080) at barrier steps
  k = 17, 18, 19 with the barrier-tied tolerance, through DeviceSystem.step (one
  kkt_dev_step call: batched refactor -> lu_solve -> lockstep FGMRES-IR with the straggler
  hand-off to single-system helpers).  EVERY system against the C oracle (the restatement of
  refactorize / lu_solve / refine_fgmres pinned to the reference's goldens): trigger equal,
  iterations within +-1, true rr within tests/large_golden.rr_bound, converged.
* The sequence: systems k = 1..19 of the same pattern, single-system handle, each against the
  oracle under the same bars (configs[2], the per-system latency line of bench.py).
* The hand-off itself at small size against the REFERENCE's goldens with several concurrent
  helpers (KKT_HANDOFF=4 on a 20-system batch).
"""

import numpy as np
import pytest

from large_golden import CASES, M, available, barrier_delta, check_report, load, rr_bound, sequence

pytestmark = pytest.mark.gpu

_PAT = {}


def _setup(config):
    if config not in _PAT:
        import bench
        from paper_2401_13926_b200 import factorize, to_general
        from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_values
        _PAT.clear()
        pat = build_pattern(ACOPF_CONFIGS[config], 0)
        K0 = pat.K.with_values(system_values(pat, 0, 0))
        f, _ = factorize(to_general(K0))
        of, ex = bench.oracle_factors(f, K0)
        _PAT[config] = (pat, f, of, ex)
    return _PAT[config]


def _oracle_run(pat, of, ex, vals, r, delta):
    from oracle import oracle
    of.refactorize(vals[ex.src])
    x, rep = of.refine_fgmres(pat.K.row_ptr, pat.K.col_idx, vals, r, of.lu_solve(r), delta)
    rr = np.linalg.norm(r - oracle.spmv(pat.K.row_ptr, pat.K.col_idx, vals, x)) / np.linalg.norm(r)
    return rep, rr


def _check(got_it, got_rr, got_trig, got_conv, orep, orr, delta, tag):
    assert bool(got_trig) == bool(orep["triggered"]), tag
    assert abs(got_it - orep["iterations"]) <= 1, (tag, got_it, orep["iterations"])
    same = got_it >= orep["iterations"]
    assert got_rr <= rr_bound(orr, delta, same), (tag, got_rr, orr)
    assert bool(got_conv) == bool(orep["converged"]), tag
    assert got_conv, tag


@pytest.mark.parametrize("k", [17, 18, 19])
def test_bench_batch_every_system_against_oracle(k):
    import bench
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200.device import DeviceSystem
    from paper_2401_13926_b200.refine import BarrierTiedTolerance
    pat, f, of, ex = _setup("activsg10k")
    B = 64
    vals, rhs, mu = bench.make_batch(pat, B, k, seed_base=bench.rank_seed_base(0))
    delta = BarrierTiedTolerance()(mu)
    dev = DeviceSystem(f, batch=B)
    torch = dev.torch
    with torch.cuda.stream(dev.stream):
        tv = torch.from_numpy(vals).to(dev.device)
        tr = torch.from_numpy(rhs).to(dev.device)
        tx = torch.empty_like(tr)
    reps = dev.step(tv, nat.LAYOUT_SYMMETRIC_LOWER, tr, tx, True, 10, 10, delta, stats=True)
    x = dev.d2h(tx)
    handed = sum(r.handed_off for r in reps)
    for q in range(B):
        orep, orr = _oracle_run(pat, of, ex, vals[q], rhs[q], delta)
        rr = np.linalg.norm(rhs[q] - _spmv(pat, vals[q], x[q])) / np.linalg.norm(rhs[q])
        _check(reps[q].iterations, rr, reps[q].triggered, reps[q].converged, orep, orr, delta,
               (k, q, reps[q].handed_off))
    if k == 19:  # the straggler path ran (iterations 6..23 across the batch)
        assert handed >= 1
    dev.close()


def _spmv(pat, vals, x):
    from oracle import oracle
    return oracle.spmv(pat.K.row_ptr, pat.K.col_idx, vals, x)


def test_sequence_every_system_against_oracle():
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200.acopf import MU_STEP, system_rhs, system_values
    from paper_2401_13926_b200.refine import BarrierTiedTolerance
    pat, f, of, ex = _setup("activsg10k")
    dev = f.device(restart_m=10)
    torch = dev.torch
    pol = BarrierTiedTolerance()
    for k in range(1, 20):
        vals, r = system_values(pat, k, 0), system_rhs(pat, k, 0)
        delta = pol(10.0 ** (-MU_STEP * k))
        with torch.cuda.stream(dev.stream):
            tv = torch.from_numpy(vals).to(dev.device)
            tr = torch.from_numpy(r).to(dev.device)
            tx = torch.empty_like(tr)
        rep = dev.step(tv, nat.LAYOUT_SYMMETRIC_LOWER, tr, tx, True, 10, 10, delta)
        x = dev.d2h(tx)
        orep, orr = _oracle_run(pat, of, ex, vals, r, delta)
        rr = np.linalg.norm(r - _spmv(pat, vals, x)) / np.linalg.norm(r)
        _check(rep.iterations, rr, rep.triggered, rep.converged, orep, orr, delta, k)


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
        check_report(dict(triggered=rep.triggered, iterations=rep.iterations, rr=rr,
                          converged=rep.converged), g["refine_1e-10"][k], (case, k), 1e-10)
        assert abs(rep.iterations - rep2.iterations) <= 1, k
        if not rep.triggered:
            assert np.array_equal(x[k], x2[k])
    dev.close()
