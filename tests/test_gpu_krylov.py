"""GPU: the generic FGMRES entry (krylov.py:36-216) and its device control.

* The reference's own FGMRES tests (test_krylov.py:52-158, 221-229) run unchanged in
  substance against ``paper_2401_13926_b200.fgmres``: identity / matrix / LU / host-callback
  operators, MGS, ``restart_residuals`` (est vs true at every restart), the flexible
  (alternating) preconditioner, NaN -> OperatorOutputError, happy breakdown.
* The device-controlled graph (one conditional-node CUDA graph per solve) and the
  host-stepped control run the same kernels: their results must be BITWISE equal.
* FGMRES with m larger than the handle's restart length (the workspace grows before any
  vector is staged in it) and per-system non-finite failures in a batch.
"""

import numpy as np
import pytest

from conftest import golden, lower_matrix
from paper_2401_13926_b200 import (MGS, KrylovConfig, LinearOperator, OperatorOutputError,
                                   RefinementConfig, factorize, fgmres, from_dense,
                                   lu_preconditioner, lu_solve, refactorize, refine_fgmres,
                                   to_general)

pytestmark = pytest.mark.gpu


# conftest.random_sparse / random_vector of the reference suite (tests/conftest.py:13-34)
def random_sparse(n, density, seed, diag_dominant=True):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n)) * (rng.random((n, n)) < density)
    if diag_dominant:
        M += np.diag(np.sign(np.diagonal(M) + 1e-3) * (np.abs(M).sum(axis=1) + 1.0))
    return from_dense(M)


def random_vector(n, seed):
    return np.random.default_rng(seed).standard_normal(n)


def test_exact_x0_zero_iterations():  # test_krylov.py:53-59
    n = 6
    I_op = LinearOperator.identity(n)
    b = random_vector(n, 1)
    res = fgmres(I_op, I_op, b, b, KrylovConfig(tol=1e-10))
    assert res.converged and res.iterations == 0
    assert res.est_residual_history[0] <= 1e-10


def test_perfect_preconditioner_callback():  # test_krylov.py:61-69 (M is a host callback)
    K = from_dense(np.diag([1.0, 2.0, 3.0, 4.0, 5.0]))
    f, _ = factorize(K)
    op = LinearOperator.from_matrix(K)
    pre = LinearOperator(5, lambda v: lu_solve(f, v))
    b = random_vector(5, 2)
    res = fgmres(op, pre, b, np.zeros(5), KrylovConfig(tol=1e-12))
    assert res.converged and res.iterations == 1
    assert res.precond_applications == res.iterations


def test_inexact_factor_preconditioner():  # test_krylov.py:71-88
    rng = np.random.default_rng(60)
    n = 60
    M = rng.standard_normal((n, n)) + np.diag(np.full(n, 6.0))
    K = from_dense(M)
    f, _ = factorize(from_dense(np.round(M, 3)))
    b = rng.standard_normal(n)
    x0 = lu_solve(f, b)
    tol = 1e-12
    for pre in (lu_preconditioner(f), LinearOperator(n, lambda v: lu_solve(f, v))):
        res = fgmres(LinearOperator.from_matrix(K), pre, b, x0, KrylovConfig(m=10, max_outer=10, tol=tol))
        assert res.converged and res.iterations <= 10
        rho0 = np.linalg.norm(b - M @ x0)
        assert np.linalg.norm(b - M @ res.x) <= 10 * tol * rho0


def test_estimate_nonincreasing_within_cycle():  # test_krylov.py:90-99
    K = random_sparse(40, 0.2, 5)
    cfg = KrylovConfig(m=5, max_outer=4, tol=1e-10)
    res = fgmres(LinearOperator.from_matrix(K), LinearOperator.identity(40), random_vector(40, 6),
                 np.zeros(40), cfg)
    hist = res.est_residual_history[1:]
    for c in range(0, len(hist), cfg.m):
        cycle = hist[c:c + cfg.m]
        assert all(b2 <= a * (1 + 1e-12) for a, b2 in zip(cycle, cycle[1:]))


def test_estimate_matches_true_at_restart():  # test_krylov.py:101-113 (restart_residuals)
    rng = np.random.default_rng(8)
    n = 50
    M = rng.standard_normal((n, n)) + np.diag(np.full(n, 8.0))
    res = fgmres(LinearOperator.from_matrix(from_dense(M)), LinearOperator.identity(n),
                 rng.standard_normal(n), np.zeros(n), KrylovConfig(m=4, max_outer=20, tol=1e-10))
    assert len(res.restart_residuals) >= 2
    for est, true in res.restart_residuals:
        if true > 0:
            assert abs(est - true) / true <= 1e-6
    assert res.restart_residuals[-1][1] == res.true_final_residual


def test_flexible_alternating_preconditioner():  # test_krylov.py:115-135 (callbacks K and M)
    rng = np.random.default_rng(9)
    n = 40
    B = rng.standard_normal((n, n))
    S = B @ B.T + n * np.eye(n)
    op = LinearOperator(n, lambda v: S @ v)
    state = {"k": 0}

    def alternating(v):
        state["k"] += 1
        return v / np.diagonal(S) if state["k"] % 2 else v.copy()

    b = rng.standard_normal(n)
    res = fgmres(op, LinearOperator(n, alternating), b, np.zeros(n),
                 KrylovConfig(m=10, max_outer=10, tol=1e-10))
    assert res.converged
    assert np.linalg.norm(b - S @ res.x) <= 10 * 1e-10 * np.linalg.norm(b)


def test_right_preconditioning_preserves_true_residual():  # test_krylov.py:137-151
    rng = np.random.default_rng(10)
    for s in range(5):
        n = 30
        K = random_sparse(n, 0.2, 100 + s)
        f, _ = factorize(K)
        b = rng.standard_normal(n)
        tol = 1e-10
        res = fgmres(LinearOperator.from_matrix(K), lu_preconditioner(f), b, np.zeros(n),
                     KrylovConfig(m=10, max_outer=10, tol=tol))
        assert res.converged
        assert np.linalg.norm(b - K.to_dense() @ res.x) <= 10 * tol * np.linalg.norm(b)


def test_nan_operator_aborts():  # test_krylov.py:153-158 (callback K)
    n = 4
    bad = LinearOperator(n, lambda v: v * np.nan)
    with pytest.raises(OperatorOutputError):
        fgmres(bad, LinearOperator.identity(n), np.ones(n), np.zeros(n), KrylovConfig())


def test_mgs_option():  # test_krylov.py:160-166
    K = random_sparse(30, 0.2, 11)
    res = fgmres(LinearOperator.from_matrix(K), LinearOperator.identity(30), random_vector(30, 12),
                 np.zeros(30), KrylovConfig(m=30, max_outer=3, tol=1e-10, ortho=MGS))
    assert res.converged


def test_happy_breakdown_is_convergence():  # test_krylov.py:221-229
    n = 5
    op = LinearOperator.identity(n)
    b = random_vector(n, 20)
    res = fgmres(op, op, b, np.zeros(n), KrylovConfig(tol=1e-12))
    assert res.converged and res.iterations == 1
    assert np.allclose(res.x, b, rtol=0, atol=1e-14)


def _late_system(case="acopf_small", k=19):
    g = golden(case)
    f, _ = factorize(to_general(lower_matrix(g, 0)))
    K = lower_matrix(g, k)
    refactorize(f, to_general(K))
    r = g["rhs"][k]
    return g, f, K, r, lu_solve(f, r)


def test_graph_equals_host_loop_single():
    """The conditional-node graph and the host-stepped control: same kernels, bitwise."""
    _g, f, K, r, x0 = _late_system()
    dev = f.device()
    dev.set_operator(K)
    out = []
    for host in (False, True, False):  # the second graph run replays the cached graph
        dev.h2d(dev.r, r)
        dev.h2d(dev.x0, x0)
        rep, hist, pairs = dev.fgmres_device(dev.r, dev.x0, dev.x, 10, 10, 1e-12, host_loop=host)
        out.append((dev.d2h(dev.x), rep.iterations, rep.restarts, hist, pairs))
    for o in out[1:]:
        assert np.array_equal(o[0], out[0][0])
        assert o[1:] == out[0][1:]
    assert out[0][1] > 0


def test_refine_m_larger_than_restart_m():
    """m > the handle's restart_m grows the workspace before staging."""
    _g, f, K, r, x0 = _late_system()
    f.close()
    dev = f.device(restart_m=10)
    for m in (10, 20, 12):
        x, rep = refine_fgmres(K, f, x0, r, RefinementConfig(delta_tol=1e-12, krylov=KrylovConfig(m=m)))
        assert rep.triggered and rep.converged, m
        assert np.linalg.norm(r - K.to_dense() @ x) / np.linalg.norm(r) <= 1e-11
    from paper_2401_13926_b200 import _native as nat
    vals = np.ascontiguousarray(K.values)
    xo = np.empty_like(r)
    rep = dev.step(vals, nat.LAYOUT_SYMMETRIC_LOWER, r, xo, False, 20, 10, 1e-12)
    assert rep.triggered and rep.converged


def test_batch_graph_equals_host_loop_and_nonfinite_isolated():
    """Batched refine: graph == host loop bitwise; a NaN system fails alone."""
    from paper_2401_13926_b200 import _native as nat
    from paper_2401_13926_b200.device import DeviceSystem
    g = golden("acopf_small")
    f, _ = factorize(to_general(lower_matrix(g, 0)))
    nb = 4
    dev = DeviceSystem(f, batch=nb)
    ks = [19, 18, 3, 17]
    vals = np.stack([g["K_values"][k] for k in ks])
    rhs = np.stack([g["rhs"][k] for k in ks])
    res = []
    t = dev.torch
    for host in (False, True):
        with t.cuda.stream(dev.stream):
            v_t = t.from_numpy(vals).cuda()
            r_t = t.from_numpy(rhs).cuda()
            x0_t = t.empty_like(r_t)
            x_t = t.empty_like(r_t)
        dev.refactor_batch(v_t, nat.LAYOUT_SYMMETRIC_LOWER)
        dev.solve_device(r_t, x0_t)
        reps = dev.refine_device(r_t, x0_t, x_t, 10, 10, 1e-10, host_loop=host)
        res.append((dev.d2h(x_t), [(q.iterations, q.triggered, q.converged) for q in reps]))
    assert np.array_equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1]
    assert res[0][1][2][1] == 0  # k = 3 is not refined at 1e-10
    # a NaN in system 1's values: its trigger test compares NaN (False, like refine.py:113),
    # it returns its (NaN) x0; the other systems are untouched
    bad = vals.copy()
    bad[1, 5] = np.nan
    xb = np.empty_like(rhs)
    reps = dev.step(bad, nat.LAYOUT_SYMMETRIC_LOWER, rhs, xb, False, 10, 10, 1e-10)
    assert reps[1].triggered == 0 and not np.all(np.isfinite(xb[1]))
    for q in (0, 2, 3):
        assert reps[q].nonfinite == 0 and reps[q].converged
        assert np.array_equal(xb[q], res[0][0][q])
