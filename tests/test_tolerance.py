"""The barrier-tied refinement tolerance delta(mu) = clamp(theta mu, delta_min, delta_max)
(refine.BarrierTiedTolerance; north-star extension, no reference counterpart — SURVEY.md §7
step 6 asks for two properties):

1. it reduces EXACTLY to the reference's fixed delta (refine.py:35) wherever theta mu is
   clamped: the policy value, and the whole per-system refine (trigger, iterations, x) on a
   synthetic sequence;
2. refinement work is non-decreasing as mu falls along the synthetic barrier sequence.

CPU tests drive the policy into the oracle's refine_fgmres (the restatement the device path is
checked against); the `gpu` tests run the same properties through the device harness.
"""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2401_13926_b200.refine import BarrierTiedTolerance, FixedTolerance

pos = st.floats(min_value=1e-300, max_value=1e300, allow_nan=False, allow_infinity=False)


@settings(max_examples=300, deadline=None)
@given(theta=pos, lo=st.floats(1e-16, 1e-4), span=st.floats(1.0, 1e6), mu=pos, mu2=pos)
def test_policy_clamps_and_is_monotone(theta, lo, span, mu, mu2):
    hi = lo * span
    p = BarrierTiedTolerance(theta=theta, delta_min=lo, delta_max=hi)
    d = p(mu)
    assert lo <= d <= hi
    if theta * mu >= hi:
        assert d == FixedTolerance(hi)(mu)
    if theta * mu <= lo:
        assert d == FixedTolerance(lo)(mu)
    if lo < theta * mu < hi:
        assert d == theta * mu
    a, b = sorted((mu, mu2))
    assert p(a) <= p(b)  # tighter as mu falls


def test_policy_validation():
    for bad in (dict(theta=0.0), dict(delta_min=0.0), dict(delta_min=1e-8, delta_max=1e-10)):
        with pytest.raises(ValueError):
            BarrierTiedTolerance(**bad)
    assert BarrierTiedTolerance()(None) == BarrierTiedTolerance().delta_max


def _oracle_sequence(seq, policy):
    from oracle import oracle
    from paper_2401_13926_b200 import factorize, to_general
    from paper_2401_13926_b200.sparse import expand_pattern
    K0 = seq.matrix(0)
    f, _ = factorize(to_general(K0))
    ex = expand_pattern(K0)
    arrays = dict(row_perm=f.row_perm.perm, col_perm=f.col_perm.perm, Lp=f._Lp, Li=f._Li,
                  Lx=f._Lx, Up=f._Up, Ui=f._Ui, Ux=f._Ux, Udiag=f._Udiag, so_ptr=f._so_ptr,
                  so_data=f._so_data, ap_ptr=f._ap_ptr, a_src=f._a_src, a_tgt=f._a_tgt)
    of = oracle.OracleFactors(arrays, ex.general.row_ptr)
    out = []
    for k in range(1, 20):
        K = seq.matrix(k)
        r = seq.rhs(k)
        of.refactorize(K.values[ex.src])
        x, rep = of.refine_fgmres(K.row_ptr, K.col_idx, K.values, r, of.lu_solve(r),
                                  policy(seq.mu(k)))
        out.append((rep["triggered"], rep["iterations"], x))
    return out


def test_clamped_policy_equals_fixed_on_a_sequence():
    from paper_2401_13926_b200.acopf import make_sequence
    seq = make_sequence("small", seed=0, length=20)
    hi = 1e-10
    clamped = BarrierTiedTolerance(theta=1e6, delta_min=1e-12, delta_max=hi)  # theta mu >= hi
    assert all(clamped(seq.mu(k)) == hi for k in range(20))
    a = _oracle_sequence(seq, clamped)
    b = _oracle_sequence(seq, FixedTolerance(hi))
    for (ta, ia, xa), (tb, ib, xb) in zip(a, b):
        assert ta == tb and ia == ib and np.array_equal(xa, xb)


def test_refinement_work_non_decreasing_as_mu_falls():
    from paper_2401_13926_b200.acopf import make_sequence
    seq = make_sequence("small", seed=0, length=20)
    its = [it for _, it, _ in _oracle_sequence(seq, BarrierTiedTolerance())]
    assert all(a <= b for a, b in zip(its, its[1:])), its
    assert its[-1] > 0  # the late systems do refine


@pytest.mark.gpu
def test_device_harness_properties():
    """Both properties through the device path (harness.run_refactor_ir, kkt_dev_step)."""
    from paper_2401_13926_b200.acopf import make_sequence
    from paper_2401_13926_b200.harness import run_refactor_ir
    from paper_2401_13926_b200.refine import RefinementConfig
    seq = make_sequence("activsg200", seed=0, length=20)
    mats = [seq.matrix(k) for k in range(20)]
    rhss = [seq.rhs(k) for k in range(20)]
    mus = [seq.mu(k) for k in range(20)]
    hi = 1e-10
    rows_c, _ = run_refactor_ir(mats, rhss, RefinementConfig(delta_tol=hi), mus=mus,
                                tolerance=BarrierTiedTolerance(theta=1e6, delta_min=1e-12,
                                                               delta_max=hi))
    rows_f, _ = run_refactor_ir(mats, rhss, RefinementConfig(delta_tol=hi), mus=mus,
                                tolerance=FixedTolerance(hi))
    for a, b in zip(rows_c, rows_f):
        assert (a.ir_iterations, a.rr, a.nsr_after) == (b.ir_iterations, b.rr, b.nsr_after)
    rows_b, _ = run_refactor_ir(mats, rhss, RefinementConfig(), mus=mus,
                                tolerance=BarrierTiedTolerance())
    its = [r.ir_iterations for r in rows_b[1:]]
    assert all(a <= b for a, b in zip(its, its[1:])), its
