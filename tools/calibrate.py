"""Calibration of the synthetic barrier sequence with the CPU oracle (SURVEY.md §8d gates):
FGMRES-IR iterations per barrier step k at delta = 1e-10 and with the barrier-tied delta.

    python tools/calibrate.py CONFIG [d_exp] [seeds] [ks]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_rhs, system_values
from paper_2401_13926_b200.refine import BarrierTiedTolerance

cfg = sys.argv[1]
d_exp = float(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
seeds = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ks = [int(k) for k in sys.argv[4].split(",")] if len(sys.argv) > 4 else list(range(1, 20))
t0 = time.time()
pat = build_pattern(ACOPF_CONFIGS[cfg], 0)
if d_exp is not None:
    pat.meta["d_exp"] = d_exp
args = bench.parse(["--config", cfg])
from paper_2401_13926_b200 import factorize, to_general  # noqa: E402
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
of, ex = bench.oracle_factors(f, pat.K)
print(f"{cfg} N={pat.N} d_exp={pat.meta.get('d_exp')} setup {time.time() - t0:.0f}s", flush=True)
pol = BarrierTiedTolerance()
for k in ks:
    row = []
    for q in range(seeds):
        v, r = system_values(pat, k, q), system_rhs(pat, k, q)
        mu = 10.0 ** (-0.4 * k)
        of.refactorize(v[ex.src])
        x0 = of.lu_solve(r)
        _, a = of.refine_fgmres(pat.K.row_ptr, pat.K.col_idx, v, r, x0, 1e-10)
        _, b = of.refine_fgmres(pat.K.row_ptr, pat.K.col_idx, v, r, x0, pol(mu))
        row.append((a["iterations"], a["converged"], b["iterations"], b["converged"]))
    print(k, row, f"{time.time() - t0:.0f}s", flush=True)
