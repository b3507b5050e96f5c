"""Chain task lists of the single-system grid solve (plan.cpp build_chains; CPU only).

The persistent, sync-free grid kernel (trisolve.cu k_trsv_chain) is deadlock-free exactly
when every task reads only values published by tasks earlier in its list: each warp takes its
tasks in list order and all warps are resident, so the earliest unfinished task can always
run.  kkt_plan_check builds the host plan kkt_dev_create would build (no GPU) and counts
violations of that order, plus coverage violations (a grid row published twice or never, a
chain's "internal" entry outside the chain, a chain row whose prefix task is missing).  The
device tests (test_gpu_parity / test_gpu_large / test_gpu_scale) check the numbers bitwise.
"""

import ctypes as C

import numpy as np
import pytest

from paper_2401_13926_b200 import _native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_values
from paper_2401_13926_b200.sparse import lower_map


def plan_check(K):
    """K: symmetric-lower CsMatrix -> the 8 kkt_plan_check counters."""
    G = to_general(K)
    f, _ = factorize(G)
    lm = lower_map(f._pattern_ref)
    rp = np.ascontiguousarray(f._pattern_ref.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(f._pattern_ref.col_idx, dtype=np.int64)
    out = np.zeros(8, dtype=np.int64)
    gs = np.ascontiguousarray(lm[2], dtype=np.int64)
    nat.check(nat.load().kkt_plan_check(f._sym.ptr, nat.ptr_i64(rp), nat.ptr_i64(ci), int(lm[1].size),
                                        nat.ptr_i64(gs), nat.ptr_i64(out)), "kkt_plan_check")
    return out, f


CASES = [("small", 1.0), ("activsg200", 1.0), ("activsg200", 0.95), ("activsg2000", 1.0), ("activsg10k", 1.0)]


@pytest.mark.parametrize("config,imbalance", CASES)
def test_chain_lists_are_topological_and_complete(config, imbalance):
    pat = build_pattern(ACOPF_CONFIGS[config], 0, imbalance_frac=imbalance)
    out, f = plan_check(pat.K.with_values(system_values(pat, 0, 0)))
    tasks_L, tasks_U, chains, chain_rows, longest, order_bad, cover_bad, _ = out.tolist()
    assert order_bad == 0 and cover_bad == 0, out
    assert longest <= 32
    if config != "small":  # the grid phases exist and contain chains at these sizes
        assert tasks_L > 0 and tasks_U > 0 and chains > 0 and chain_rows >= 2 * chains


def test_standard_trace_plan():
    from conftest import golden, lower_matrix
    out, _ = plan_check(lower_matrix(golden("standard_trace"), 0))
    assert out[5] == 0 and out[6] == 0, out


def test_plan_check_rejects_null():
    lib = nat.load()
    out = np.zeros(8, dtype=np.int64)
    assert lib.kkt_plan_check(None, None, None, 0, None, nat.ptr_i64(out)) == nat.KKT_ERR_BAD_ARG
