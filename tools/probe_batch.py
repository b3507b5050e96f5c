"""Batch throughput probe: refactor / solve / full step for B same-pattern systems."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import build_pattern, ACOPF_CONFIGS, system_values, system_rhs
from paper_2401_13926_b200.device import DeviceSystem

cfg = sys.argv[1] if len(sys.argv) > 1 else "activsg10k"
Bs = [int(b) for b in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 8, 32, 64]
pat = build_pattern(ACOPF_CONFIGS[cfg], 0)
f, _ = factorize(to_general(pat.K))
for B in Bs:
    dev = DeviceSystem(f, batch=B)
    ks = [1 + q % 19 for q in range(B)]
    vals = np.stack([system_values(pat, k, q // 19) for q, k in enumerate(ks)])
    rhs = np.stack([system_rhs(pat, k, q // 19) for q, k in enumerate(ks)])
    s = dev.stream
    with torch.cuda.stream(s):
        tv = torch.from_numpy(vals).to(dev.device)
        tr = torch.from_numpy(rhs).to(dev.device)
        tx = torch.empty_like(tr)
    s.synchronize()

    def timed(fn, reps=3):
        ts = []
        for _ in range(reps):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            e.record(s)
            e.synchronize()
            ts.append(a.elapsed_time(e))
        return min(ts)

    tref = timed(lambda: dev.refactor_device(tv, nat.LAYOUT_SYMMETRIC_LOWER))
    tsol = timed(lambda: dev.solve_device(tr, tx))
    its = []

    def step():
        reps = dev.step(tv, nat.LAYOUT_SYMMETRIC_LOWER, tr, tx, True, 10, 10, 1e-10)
        its.append(np.mean([r.iterations for r in (reps if B > 1 else [reps])]))

    tstep = timed(step)
    print(f"B={B:3d} refactor {tref:8.3f} ms ({tref / B:7.3f}/sys)  solve {tsol:8.3f} ms ({tsol / B:7.3f}/sys)  "
          f"step {tstep:8.3f} ms ({tstep / B:7.3f}/sys) mean IR its {its[-1]:.2f}", flush=True)
    dev.close()
    del tv, tr, tx
    torch.cuda.empty_cache()
