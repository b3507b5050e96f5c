"""Per-config measurements (BASELINE.json configs[0..4]) on one B200: single-system
sequence latency (refactor + solve + FGMRES-IR, barrier-tied tolerance, L2 flushed before
each system) and, where given, batched throughput.  Prints one JSON line per config.
usage: bench_configs.py activsg200 activsg2000 activsg10k activsg70k [--batch B]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, MU_STEP, build_pattern, system_rhs, system_values
from paper_2401_13926_b200.refine import BarrierTiedTolerance

LOWER = nat.LAYOUT_SYMMETRIC_LOWER
policy = BarrierTiedTolerance()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for cfg in [a for a in sys.argv[1:] if not a.startswith("--")]:
    t0 = time.perf_counter()
    pat = build_pattern(ACOPF_CONFIGS[cfg], 0)
    f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
    analyze_s = time.perf_counter() - t0
    dev = f.device(restart_m=10)
    M = 20
    lat, its, ref_ms, sol_ms = [], [], [], []
    for k in range(1, M):
        with torch.cuda.stream(dev.stream):
            v = torch.from_numpy(system_values(pat, k, 0)).to(dev.device)
            r = torch.from_numpy(system_rhs(pat, k, 0)).to(dev.device)
            x = torch.empty_like(r)
        for what in ("step", "refactor", "solve"):
            with torch.cuda.stream(dev.stream):
                flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(dev.stream)
            if what == "step":
                rep = dev.step(v, LOWER, r, x, True, 10, 10, policy(10.0 ** (-MU_STEP * k)))
            elif what == "refactor":
                dev.refactor_device(v, LOWER)
            else:
                dev.solve_device(r, x)
            b.record(dev.stream)
            b.synchronize()
            {"step": lat, "refactor": ref_ms, "solve": sol_ms}[what].append(a.elapsed_time(b))
        its.append(rep.iterations)
    st = f.stats
    print(json.dumps({"config": cfg, "N": pat.N, "nnz_lower": int(pat.K.nnz), "nnz_L": st["nnz_L"],
                      "nnz_U": st["nnz_U"], "levels": st["refactor_levels"],
                      "update_pairs": st["update_pairs"], "analyze_s": round(analyze_s, 2),
                      "single_ms_per_system_mean": float(np.mean(lat)),
                      "single_ms_median": float(np.median(lat)),
                      "refactor_ms_median": float(np.median(ref_ms)),
                      "trisolve_pair_ms_median": float(np.median(sol_ms)), "ir_iterations": its}),
          flush=True)
    dev.close()
