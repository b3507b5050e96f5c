"""pipeline.BatchPipeline (the e2e path of bench.py): streamed batches with the values / rhs
uploads, the refactorization and the solution downloads overlapped on two streams give the
same solutions (bitwise) and FGMRES reports as one synchronous kkt_dev_step per batch."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_pipeline_matches_step():
    import torch
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200 import factorize, to_general
    from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, MU_STEP, build_pattern, system_rhs, system_values
    from paper_2401_13926_b200.device import DeviceSystem
    from paper_2401_13926_b200.pipeline import BatchPipeline, as_pinned
    from paper_2401_13926_b200.refine import BarrierTiedTolerance
    pat = build_pattern(ACOPF_CONFIGS["activsg200"], 0)
    f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
    B, LOWER, pol = 8, nat.LAYOUT_SYMMETRIC_LOWER, BarrierTiedTolerance()
    batches = []
    for s, k in enumerate([3, 17, 11, 19]):  # late barrier steps trigger FGMRES
        ks = [1 + (k + q) % 19 for q in range(B)]
        vals = np.stack([system_values(pat, kk, q) for q, kk in enumerate(ks)])
        rhs = np.stack([system_rhs(pat, kk, q) for q, kk in enumerate(ks)])
        delta = [pol(10.0 ** (-MU_STEP * kk)) for kk in ks]
        batches.append((vals, rhs, delta))
    dev = DeviceSystem(f, batch=B)
    items = [(as_pinned(v), as_pinned(r), torch.empty(r.shape, dtype=torch.float64).pin_memory(), dl)
             for v, r, dl in batches]
    reps = BatchPipeline(dev, LOWER).run(items)
    ref = DeviceSystem(f, batch=B)
    for (v, r, dl), it, rp in zip(batches, items, reps):
        x = np.empty_like(r)
        rr = ref.step(v, LOWER, r, x, False, 10, 10, dl)
        assert np.array_equal(it[2].numpy(), x)
        assert [q.iterations for q in rp] == [q.iterations for q in rr]
        assert [bool(q.triggered) for q in rp] == [bool(q.triggered) for q in rr]
    assert any(q.iterations > 0 for rp in reps for q in rp)
    dev.close()
    ref.close()
