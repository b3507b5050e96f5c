"""Kernel probe: time refactor / trisolve / spmv on one config (used with ncu launch lists)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import make_sequence

cfg = sys.argv[1] if len(sys.argv) > 1 else "activsg10k"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
seq = make_sequence(cfg, seed=0, length=20)
f, _ = factorize(to_general(seq.matrix(0)))
dev = f.device()
print(dev.info())
s = dev.stream
with torch.cuda.stream(s):
    vals = torch.from_numpy(seq.values(19)).cuda()
    b = torch.randn(seq.pattern.N, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
s.synchronize()
for name, fn in [("refactor", lambda: dev.refactor_device(vals, nat.LAYOUT_SYMMETRIC_LOWER)),
                 ("solve", lambda: dev.solve_device(b, x)),
                 ("spmv", lambda: dev.spmv_device(b, x))]:
    ts = []
    for _ in range(reps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        e.record(s)
        e.synchronize()
        ts.append(a.elapsed_time(e))
    print(name, [round(t, 4) for t in ts])
