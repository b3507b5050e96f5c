"""A small workload that drives every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

* single-system handle: refactorize -> lu_solve -> refine_fgmres (graph control) on the
  acopf_small golden's late systems, plus the host-stepped control;
* batched handle (nb = 33, KKT_B_SPLIT_NP=8 so the wide columns take the TMA pipeline):
  refactor, solve, SpMV, lockstep FGMRES-IR with the straggler hand-off (KKT_HANDOFF=4).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("KKT_B_SPLIT_NP", "8")
os.environ.setdefault("KKT_HANDOFF", "4")

import numpy as np  # noqa: E402

from conftest import golden, lower_matrix  # noqa: E402
import paper_2401_13926_b200._native as nat  # noqa: E402
from paper_2401_13926_b200 import factorize, to_general  # noqa: E402
from paper_2401_13926_b200.device import DeviceSystem  # noqa: E402

g = golden("acopf_small")
M = g["K_values"].shape[0]
f, _ = factorize(to_general(lower_matrix(g, 0)))
LOWER = nat.LAYOUT_SYMMETRIC_LOWER
dev = f.device(restart_m=10)
for k in (M - 2, M - 1):
    x = np.empty_like(g["rhs"][k])
    rep = dev.step(np.ascontiguousarray(g["K_values"][k]), LOWER, g["rhs"][k], x, False, 10, 10,
                   1e-10, stats=True)
    print("single", k, rep.iterations, rep.converged)
dev.close()
nb = 33
systems = [(M - 1 - q) % M for q in range(nb)]
vals = np.ascontiguousarray(np.stack([g["K_values"][k] for k in systems]))
rhs = np.ascontiguousarray(np.stack([g["rhs"][k] for k in systems]))
devb = DeviceSystem(f, batch=nb)
x = np.empty_like(rhs)
reps = devb.step(vals, LOWER, rhs, x, False, 10, 10, [1e-10] * nb, stats=True)
print("batch", [r.iterations for r in reps], sum(r.handed_off for r in reps))
devb.close()
print("sanitize case done")
