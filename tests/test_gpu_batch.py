"""Batched handle (nb same-pattern systems in one launch sequence) vs the reference.

Every system of a batch must reproduce the reference exactly like the single-system path:
refactorized factors and lu_solve bitwise, FGMRES-IR trigger equal and iterations within
+-1 (the 64-system configuration of BASELINE.json)."""

import numpy as np
import pytest

from conftest import golden, lower_matrix
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200 import _native as nat

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case,nb,env", [
    ("acopf_small", 5, {}), ("standard_trace", 9, {}), ("acopf_tiny", 20, {}),
    ("acopf_small", 40, {"KKT_B_HEAVY_NP": "8"}), ("standard_trace", 3, {"KKT_B_HEAVY_NP": "4"}),
    ("acopf_small", 33, {"KKT_B_SPLIT_NP": "8"}), ("standard_trace", 9, {"KKT_B_SPLIT_NP": "4"}),
    ("acopf_small", 7, {"KKT_B_SPLIT_NP": "8", "KKT_B_HEAVY_NP": "16"}),
    ("acopf_small", 33, {"KKT_B_SPLIT_NP": "8", "KKT_B_CT_MODE": "1"}),
    ("standard_trace", 9, {"KKT_B_SPLIT_NP": "4", "KKT_B_CT_MODE": "1", "KKT_B_CT_SC": "4"}),
    ("acopf_small", 33, {"KKT_B_SPLIT_NP": "8", "KKT_B_CT_MODE": "0"}),
    ("acopf_small", 33, {"KKT_B_SPLIT_NP": "8", "KKT_B_TMA_DIRECT": "0", "KKT_B_TMA": "4,128"}),
    ("standard_trace", 9, {"KKT_B_SPLIT_NP": "4", "KKT_B_TMA": "3,160"}),
    ("acopf_small", 33, {"KKT_B_SPLIT_NP": "8", "KKT_B_TAIL_ORDER": "1"}),
    ("acopf_small", 33, {"KKT_B_SPLIT_NP": "8", "KKT_B_TMA_DIRECT": "1"}),
    ("acopf_small", 33, {"KKT_B_SPLIT_NP": "8", "KKT_B_TMA_E": "64"}),
    # one system per lane in the light-column replay (k_b_refactor; default: two per lane)
    ("acopf_small", 33, {"KKT_B_V2": "0"}), ("standard_trace", 9, {"KKT_B_V2": "0"}),
    # flag-free wide-column producer (default with the 128-row ring: 70k-class patterns)
    ("acopf_small", 33, {"KKT_B_SPLIT_NP": "8", "KKT_B_TMA_DIRECT": "3"}),
    ("acopf_small", 40, {"KKT_B_SPLIT_NP": "8", "KKT_B_TMA": "2,128"}),
    ("standard_trace", 9, {"KKT_B_SPLIT_NP": "4", "KKT_B_TMA": "2,128", "KKT_B_TMA_DIRECT": "2"}),
    # solve variants: grid-solve (chunk, CTAs/SM), sweep look-ahead / width, U head prefix
    ("acopf_small", 33, {"KKT_B_GRIDV": "0"}), ("standard_trace", 9, {"KKT_B_GRIDV": "1"}),
    ("acopf_small", 40, {"KKT_B_GRIDV": "2"}), ("acopf_small", 33, {"KKT_B_GRIDV": "4"}),
    ("acopf_small", 33, {"KKT_SWEEP_AHEAD": "1"}), ("standard_trace", 9, {"KKT_SWEEP_AHEAD": "1"}),
    ("acopf_small", 33, {"KKT_SWEEP_THREADS": "512"}), ("acopf_small", 33, {"KKT_U_PARTIAL": "0"}),
    ("acopf_small", 33, {"KKT_B_SPMV_TILES": "1"})])
def test_batch_refactor_solve_bitwise(case, nb, env, monkeypatch):
    """env forces the alternative replay kernels onto small cases: KKT_B_SPLIT_NP (4-warp CTA
    tasks for the wide columns), KKT_B_HEAVY_NP (pull-form CTA per 32 systems)."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    from paper_2401_13926_b200.device import DeviceSystem
    g = golden(case)
    M = g["K_values"].shape[0]
    systems = [(M - 1 - q) % M for q in range(nb)]  # mixed order incl. repeats when nb > M
    f, _ = factorize(to_general(lower_matrix(g, 0)))
    dev = DeviceSystem(f, batch=nb)
    vals = np.ascontiguousarray(np.stack([g["K_values"][k] for k in systems]))
    rhs = np.ascontiguousarray(np.stack([g["rhs"][k] for k in systems]))
    with torch.cuda.stream(dev.stream):
        tv = torch.from_numpy(vals).to(dev.device)
        tr = torch.from_numpy(rhs).to(dev.device)
        tx = torch.empty_like(tr)
    diag = dev.refactor_batch(tv, nat.LAYOUT_SYMMETRIC_LOWER)
    Lx, Ux, Ud = dev.download_factors_batch()
    dev.solve_device(tr, tx)
    x = dev.d2h(tx)
    for q, k in enumerate(systems):
        assert np.array_equal(diag[q], g["refactor_diag"][k]), (q, k)
        if f"s{k}_Lx" in g:
            assert np.array_equal(Lx[q], g[f"s{k}_Lx"]), (q, k)
            assert np.array_equal(Ux[q], g[f"s{k}_Ux"]), (q, k)
            assert np.array_equal(Ud[q], g[f"s{k}_Udiag"]), (q, k)
        assert np.array_equal(x[q], g["x0"][k]), (q, k)
    dev.close()


@pytest.mark.parametrize("case,nb", [("acopf_small", 6), ("standard_trace", 9)])
def test_batch_step_matches_reference(case, nb):
    import torch
    from paper_2401_13926_b200.device import DeviceSystem
    g = golden(case)
    M = g["K_values"].shape[0]
    systems = [M - 1 - q for q in range(nb)]
    ref = g["refine_1e-10_report"]
    f, _ = factorize(to_general(lower_matrix(g, 0)))
    dev = DeviceSystem(f, batch=nb)
    vals = np.ascontiguousarray(np.stack([g["K_values"][k] for k in systems]))
    rhs = np.ascontiguousarray(np.stack([g["rhs"][k] for k in systems]))
    x = np.empty_like(rhs)
    reps = dev.step(vals, nat.LAYOUT_SYMMETRIC_LOWER, rhs, x, False, 10, 10, 1e-10)
    for q, k in enumerate(systems):
        K = lower_matrix(g, k)
        assert bool(reps[q].triggered) == bool(ref[k, 0]), (q, k)
        assert abs(reps[q].iterations - int(ref[k, 1])) <= 1, (q, k, reps[q].iterations, ref[k, 1])
        assert reps[q].converged
        rr = np.linalg.norm(rhs[q] - K.to_dense() @ x[q]) / np.linalg.norm(rhs[q])
        xr = g["refine_1e-10_x"][k]
        rr_ref = np.linalg.norm(rhs[q] - K.to_dense() @ xr) / np.linalg.norm(rhs[q])
        assert rr <= max(1.5 * rr_ref, 4 * np.finfo(float).eps), (q, k, rr, rr_ref)
    dev.close()


@pytest.mark.parametrize("tiles", ["0", "1"])
@pytest.mark.parametrize("case,nb", [("acopf_small", 33), ("standard_trace", 9), ("acopf_tiny", 40)])
def test_batch_spmv_residual_and_norms_bitwise(case, nb, tiles, monkeypatch):
    """The batched SpMV (per-row kernel, and the tiled flat walk with KKT_B_SPMV_TILES=1),
    residual statistics and the tiled value expansion against the reference's spmv
    (sparsecore.py:284-305) and inf_norm: every system bitwise."""
    import torch
    monkeypatch.setenv("KKT_B_SPMV_TILES", tiles)
    from oracle import oracle
    from paper_2401_13926_b200.device import DeviceSystem
    from paper_2401_13926_b200.sparse import to_general
    g = golden(case)
    M = g["K_values"].shape[0]
    systems = [(M - 1 - q) % M for q in range(nb)]
    f, _ = factorize(to_general(lower_matrix(g, 0)))
    dev = DeviceSystem(f, batch=nb)
    vals = np.ascontiguousarray(np.stack([g["K_values"][k] for k in systems]))
    x0 = np.ascontiguousarray(np.stack([g["x0"][k] for k in systems]))
    rhs = np.ascontiguousarray(np.stack([g["rhs"][k] for k in systems]))
    with torch.cuda.stream(dev.stream):
        tv = torch.from_numpy(vals).to(dev.device)
        tx = torch.from_numpy(x0).to(dev.device)
        tr = torch.from_numpy(rhs).to(dev.device)
        ty = torch.empty_like(tx)
    dev.refactor_batch(tv, nat.LAYOUT_SYMMETRIC_LOWER)
    dev.spmv_device(tx, ty)
    y = dev.d2h(ty)
    stats = dev.residual_stats_device(tr, tx)
    for q, k in enumerate(systems):
        assert np.array_equal(y[q], g["spmv_K_x0"][k]), (q, k)
        K = lower_matrix(g, k)
        e = rhs[q] - g["spmv_K_x0"][k]
        assert stats[q].err_inf == np.max(np.abs(e)), (q, k)
        assert stats[q].k_inf == oracle.inf_norm(K.row_ptr, K.col_idx, K.values), (q, k)
    dev.close()
