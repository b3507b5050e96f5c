"""Parity at the BASELINE.json sizes (configs[0..4]): the device path against the C oracle
(oracle/kkt_oracle.c, the restatement of direct_lu.refactorize / lu_solve and
refine.refine_fgmres, pinned to the reference's golden vectors by test_oracle.py) on the
same ACOPF-shaped sequences the bench uses.

* refactorize: factor values bitwise equal to the oracle's (late, ill-conditioned system);
* lu_solve: bitwise;
* refine_fgmres: trigger equal, iterations within +-1, final relative residual within
  max(1.5 x oracle, 4 eps) (SURVEY.md §7 hard part 5) — checked with the oracle's SpMV;
* batch of 4 systems (interleaved handle): every system bitwise equal to its single-system
  factors / solution (and so to the oracle).
"""

import numpy as np
import pytest

from large_golden import rr_floor

pytestmark = pytest.mark.gpu

CONFIGS = [("activsg200", 19), ("activsg2000", 19), ("activsg10k", 19),
           ("activsg10k/0.95", 19),  # the off-diagonal pivoting regime at 238k (4,214 pivots)
           ("activsg10k/0.9", 19),   # 8,336 pivots, 390M update pairs per refactorization
           pytest.param("activsg70k", 19, marks=pytest.mark.slow)]


def _setup(config):
    from paper_2401_13926_b200 import factorize, to_general
    from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_values
    config, _, frac = config.partition("/")
    pat = build_pattern(ACOPF_CONFIGS[config], 0, imbalance_frac=float(frac or 1.0))
    K0 = pat.K.with_values(system_values(pat, 0, 0))
    f, _ = factorize(to_general(K0))
    return pat, K0, f


def _oracle(f, K0):
    from oracle import oracle
    from paper_2401_13926_b200.sparse import expand_pattern
    ex = expand_pattern(K0)
    arrays = dict(row_perm=f.row_perm.perm, col_perm=f.col_perm.perm, Lp=f._Lp, Li=f._Li,
                  Lx=f._Lx, Up=f._Up, Ui=f._Ui, Ux=f._Ux, Udiag=f._Udiag, so_ptr=f._so_ptr,
                  so_data=f._so_data, ap_ptr=f._ap_ptr, a_src=f._a_src, a_tgt=f._a_tgt)
    return oracle.OracleFactors(arrays, ex.general.row_ptr), ex


@pytest.mark.parametrize("config,k", CONFIGS)
def test_full_size_against_oracle(config, k):
    import torch
    from oracle import oracle
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200.acopf import MU_STEP, system_rhs, system_values
    from paper_2401_13926_b200.refine import BarrierTiedTolerance
    pat, K0, f = _setup(config)
    if "/" in config:  # row_perm != col_perm (direct_lu.py:209-223)
        assert f.stats["offdiag_pivots"] > 0
    of, ex = _oracle(f, K0)
    vals = system_values(pat, k, 0)
    r = system_rhs(pat, k, 0)
    delta = BarrierTiedTolerance()(10.0 ** (-MU_STEP * k))
    # oracle
    of.refactorize(vals[ex.src])
    ox0 = of.lu_solve(r)
    ox, orep = of.refine_fgmres(pat.K.row_ptr, pat.K.col_idx, vals, r, ox0, delta)
    # device, single system
    dev = f.device(restart_m=10)
    LOWER = nat.LAYOUT_SYMMETRIC_LOWER
    with torch.cuda.stream(dev.stream):
        tv = torch.from_numpy(vals).to(dev.device)
        tr = torch.from_numpy(r).to(dev.device)
        tx = torch.empty_like(tr)
    dev.refactor_device(tv, LOWER)
    Lx, Ux, Ud = dev.download_factors()
    assert np.array_equal(Lx, of.a["Lx"]) and np.array_equal(Ux, of.a["Ux"])
    assert np.array_equal(Ud, of.a["Udiag"])
    dev.solve_device(tr, tx)
    x0 = dev.d2h(tx)
    assert np.array_equal(x0, ox0)
    rep = dev.step(tv, LOWER, tr, tx, True, 10, 10, delta)
    x = dev.d2h(tx)
    assert bool(rep.triggered) == orep["triggered"]
    assert abs(rep.iterations - orep["iterations"]) <= 1, (rep.iterations, orep["iterations"])
    nr = np.linalg.norm(r)
    rr = np.linalg.norm(r - oracle.spmv(pat.K.row_ptr, pat.K.col_idx, vals, x)) / nr
    rr_o = np.linalg.norm(r - oracle.spmv(pat.K.row_ptr, pat.K.col_idx, vals, ox)) / nr
    assert rr <= max(1.5 * rr_o, 4 * np.finfo(float).eps), (rr, rr_o)


@pytest.mark.parametrize("config,nb", [("activsg200", 4), ("activsg10k", 4), ("activsg2000", 40),
                                       ("activsg10k/0.95", 4), ("activsg10k/0.9", 4),
                                       ("activsg10k/ring128", 8),
                                       pytest.param("activsg70k", 8, marks=pytest.mark.slow)])
def test_full_size_batch_equals_single(config, nb, monkeypatch):
    """The interleaved batch reproduces each system's single-system factors and solve (nb = 40:
    8-system groups of the TMA wide-column pipeline, every group's done flags and the
    padding systems of the last 32-block; ring128: the 128-row stage ring with the flag-free
    producer, the default for 70k-class patterns, forced at 10k)."""
    import torch
    if config.endswith("/ring128"):
        config = config[:-len("/ring128")]
        monkeypatch.setenv("KKT_B_TMA", "2,128")
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200.acopf import system_rhs, system_values
    from paper_2401_13926_b200.device import DeviceSystem
    pat, K0, f = _setup(config)
    ks = [3, 11, 17, 19] if nb == 4 else [1 + (7 * q) % 19 for q in range(nb)]
    vals = np.stack([system_values(pat, k, q % 4) for q, k in enumerate(ks)])
    rhs = np.stack([system_rhs(pat, k, q % 4) for q, k in enumerate(ks)])
    LOWER = nat.LAYOUT_SYMMETRIC_LOWER
    devb = DeviceSystem(f, batch=len(ks))
    with torch.cuda.stream(devb.stream):
        tv = torch.from_numpy(vals).to(devb.device)
        tr = torch.from_numpy(rhs).to(devb.device)
        tx = torch.empty_like(tr)
    devb.refactor_batch(tv, LOWER)
    Lb, Ub, Db = devb.download_factors_batch()
    devb.solve_device(tr, tx)
    xb = devb.d2h(tx)
    dev1 = f.device(restart_m=10)
    for q in range(len(ks)):
        with torch.cuda.stream(dev1.stream):
            v1 = torch.from_numpy(vals[q]).to(dev1.device)
            r1 = torch.from_numpy(rhs[q]).to(dev1.device)
            x1 = torch.empty_like(r1)
        dev1.refactor_device(v1, LOWER)
        L1, U1, D1 = dev1.download_factors()
        assert np.array_equal(Lb[q], L1) and np.array_equal(Ub[q], U1) and np.array_equal(Db[q], D1)
        dev1.solve_device(r1, x1)
        assert np.array_equal(xb[q], dev1.d2h(x1))
    devb.close()


def _oracle_refine_all(f, K0, pat, items, threads=8):
    """Oracle refactorize + lu_solve + refine_fgmres of every (values, rhs, delta) item,
    one OracleFactors per worker thread (the C oracle releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle
    out = [None] * len(items)

    def work(w):
        of, ex = _oracle(f, K0)
        for i in range(w, len(items), threads):
            vals, r, delta = items[i]
            of.refactorize(vals[ex.src])
            x0 = of.lu_solve(r)
            x, rep = of.refine_fgmres(pat.K.row_ptr, pat.K.col_idx, vals, r, x0, delta)
            rr = np.linalg.norm(r - oracle.spmv(pat.K.row_ptr, pat.K.col_idx, vals, x)) / np.linalg.norm(r)
            out[i] = (x0, rep, rr)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    return out


def _check_vs_oracle(tag, rep, rr, orep, rr_o, delta, floor=0.0):
    from large_golden import rr_bound
    assert bool(rep.triggered) == orep["triggered"], tag
    assert abs(rep.iterations - orep["iterations"]) <= 1, (tag, rep.iterations, orep["iterations"])
    assert bool(rep.converged) == orep["converged"] and rep.converged, tag
    assert rr <= rr_bound(rr_o, delta, rep.iterations >= orep["iterations"], floor), (tag, rr, rr_o, floor)


def test_bench_batch_against_oracle():
    """The benchmarked configuration itself: bench.py's B = 64 batch at ACTIVSg10k (its value
    streams, barrier-tied delta) through the exact call the bench times (kkt_dev_step on the
    device-resident batch), at the three latest (most refined) barrier steps k = 17, 18, 19;
    every one of the 192 systems against the oracle."""
    import torch
    import paper_2401_13926_b200._native as nat
    from bench import make_batch, shard
    from paper_2401_13926_b200.device import DeviceSystem
    from paper_2401_13926_b200.refine import BarrierTiedTolerance
    pat, K0, f = _setup("activsg10k")
    B = 64
    dev = DeviceSystem(f, restart_m=10, batch=B)
    LOWER = nat.LAYOUT_SYMMETRIC_LOWER
    policy = BarrierTiedTolerance()
    for k in (17, 18, 19):
        vals, rhs, mu = make_batch(pat, shard(0, 1, B, "strong"), k)
        delta = policy(mu)
        with torch.cuda.stream(dev.stream):
            tv = torch.from_numpy(vals).to(dev.device)
            tr = torch.from_numpy(rhs).to(dev.device)
            tx = torch.empty_like(tr)
        reps = dev.step(tv, LOWER, tr, tx, True, 10, 10, [delta] * B, stats=True)
        x = dev.d2h(tx)
        ores = _oracle_refine_all(f, K0, pat, [(vals[q], rhs[q], delta) for q in range(B)])
        for q in range(B):
            x0, orep, rr_o = ores[q]
            rep = reps[q]
            rr = rep.stats_after[0] / rep.stats_after[4] if rep.triggered else \
                rep.stats_before[0] / rep.stats_before[4]
            fl = rr_floor(pat.K.row_ptr, pat.K.col_idx, vals[q], x[q], rhs[q])
            _check_vs_oracle((k, q, rep.handed_off), rep, rr, orep, rr_o, delta, fl)
            if not rep.triggered:
                assert np.array_equal(x[q], x0), (k, q)
        if k == 19:  # iterations 6..23 across the batch: the stragglers finish on helpers
            assert sum(r.handed_off for r in reps) >= 1
    dev.close()


def test_sequence_238k_against_oracle():
    """The north-star sequence (configs[2]): systems 1..19 of the ACTIVSg10k barrier sequence
    one at a time on a single-system handle, each against the oracle (factors and x0 bitwise,
    refine within the bars)."""
    import torch
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200.acopf import MU_STEP, system_rhs, system_values
    from paper_2401_13926_b200.refine import BarrierTiedTolerance
    pat, K0, f = _setup("activsg10k")
    policy = BarrierTiedTolerance()
    items = [(system_values(pat, k, 0), system_rhs(pat, k, 0), policy(10.0 ** (-MU_STEP * k)))
             for k in range(1, 20)]
    ores = _oracle_refine_all(f, K0, pat, items)
    dev = f.device(restart_m=10)
    LOWER = nat.LAYOUT_SYMMETRIC_LOWER
    for i, (vals, r, delta) in enumerate(items):
        with torch.cuda.stream(dev.stream):
            tv = torch.from_numpy(vals).to(dev.device)
            tr = torch.from_numpy(r).to(dev.device)
            tx = torch.empty_like(tr)
        dev.solve_device(tr, tx)  # warm path; the step below refactorizes first
        rep = dev.step(tv, LOWER, tr, tx, True, 10, 10, delta, stats=True)
        fl = rr_floor(pat.K.row_ptr, pat.K.col_idx, vals, dev.d2h(tx), r)
        x0_o, orep, rr_o = ores[i]
        dev.solve_device(tr, tx)
        assert np.array_equal(dev.d2h(tx), x0_o), i + 1  # factors of system i+1 -> x0 bitwise
        rr = rep.stats_after[0] / rep.stats_after[4] if rep.triggered else \
            rep.stats_before[0] / rep.stats_before[4]
        _check_vs_oracle(i + 1, rep, rr, orep, rr_o, delta, fl)
