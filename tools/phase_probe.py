"""Phase timings of one handle: refactor, lu_solve pair, SpMV (CUDA events, L2 flushed before
each rep, median of reps).  B = 1 uses the single-system handle.  Prints one JSON line per B.

    python tools/phase_probe.py CONFIG B1,B2,... [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_rhs, system_values
from paper_2401_13926_b200.device import DeviceSystem

cfg = sys.argv[1]
Bs = [int(b) for b in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
pat = build_pattern(ACOPF_CONFIGS[cfg], 0, imbalance_frac=float(os.environ.get("IMBALANCE_FRAC", "1.0")))
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
LOWER = nat.LAYOUT_SYMMETRIC_LOWER
for B in Bs:
    dev = f.device(restart_m=10) if B == 1 else DeviceSystem(f, batch=B)
    ks = [1 + q % 19 for q in range(B)]
    vals = np.stack([system_values(pat, k, q) for q, k in enumerate(ks)])
    rhs = np.stack([system_rhs(pat, k, q) for q, k in enumerate(ks)])
    if B == 1:
        vals, rhs = vals[0], rhs[0]
    s = dev.stream
    with torch.cuda.stream(s):
        tv = torch.from_numpy(vals).to(dev.device)
        tr = torch.from_numpy(rhs).to(dev.device)
        tx = torch.empty_like(tr)
    s.synchronize()

    def timed(fn, cold=True):
        ts = []
        for _ in range(reps):
            if cold:
                with torch.cuda.stream(s):
                    flush.fill_(1.0)
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            e.record(s)
            e.synchronize()
            ts.append(a.elapsed_time(e))
        return round(float(np.median(ts)), 4)

    ref = (lambda: dev.refactor_device(tv, LOWER)) if B == 1 else (lambda: dev.refactor_batch(tv, LOWER))
    out = {"config": cfg, "B": B, "env": {k: v for k, v in os.environ.items() if k.startswith("KKT_")},
           "refactor_ms": timed(ref), "solve_ms": timed(lambda: dev.solve_device(tr, tx)),
           "spmv_ms": timed(lambda: dev.spmv_device(tr, tx))}
    out["solve_warm_ms"] = timed(lambda: dev.solve_device(tr, tx), cold=False)
    out["refactor_then_solve_ms"] = timed(lambda: (ref(), dev.solve_device(tr, tx)))
    if B == 1:
        from paper_2401_13926_b200.acopf import MU_STEP
        from paper_2401_13926_b200.refine import BarrierTiedTolerance
        for k in (1, 19):
            with torch.cuda.stream(s):
                vk = torch.from_numpy(system_values(pat, k, 0)).to(dev.device)
                rk = torch.from_numpy(system_rhs(pat, k, 0)).to(dev.device)
            d = BarrierTiedTolerance()(10.0 ** (-MU_STEP * k))
            it = []
            out[f"step_k{k}_ms"] = timed(lambda: it.append(dev.step(vk, LOWER, rk, tx, True, 10, 10, d).iterations))
            out[f"step_k{k}_iters"] = it[-1]
    out["refactor_per_sys"] = round(out["refactor_ms"] / B, 4)
    out["solve_per_sys"] = round(out["solve_ms"] / B, 4)
    print(json.dumps(out), flush=True)
    dev.close()
