"""Timeline of the blocked sweeps (KKT_TRACE=1, single system): per-block phase durations."""
import ctypes as C
import os
import sys

os.environ["KKT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_rhs, system_values
from paper_2401_13926_b200.device import DeviceSystem

pat = build_pattern(ACOPF_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "activsg10k"], 0)
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
dev = DeviceSystem(f)
with torch.cuda.stream(dev.stream):
    tr = torch.from_numpy(system_rhs(pat, 1, 0)).to(dev.device)
    tx = torch.empty_like(tr)
for _ in range(3):
    dev.solve_device(tr, tx)
dev.sync()
n = f.n
ref = np.zeros(2 * n, dtype=np.uint64)
tri = np.zeros(2 * n, dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace(dev.h, ref.ctypes.data_as(C.c_void_p), tri.ctypes.data_as(C.c_void_p)))
info = dev.info()
# the sweeps write {top, tiles ready, y ready, end} per block at trace_trsv + (U ? n : 0) + p + 4 c
for name, T, off in (("L", info["L_tail_rows"], info["pL"]), ("U", info["U_head_rows"], n + info["pU"])):
    nb = (T + 31) // 32
    t = tri[off:off + 4 * nb].astype(np.int64).reshape(nb, 4)
    if not t.any():
        continue
    d = np.diff(t, axis=1)
    blk = np.diff(t[:, 0])
    print(f"{name}: blocks {nb}, total {(t[-1, 3] - t[0, 0]) / 1e3:.1f} us; mean per block: "
          f"wait+tiles {d[:, 0].mean():.0f} ns, chain {d[:, 1].mean():.0f} ns, publish+stage+B {d[:, 2].mean():.0f} ns, "
          f"top->top {blk.mean():.0f} ns; max phase B {d[:, 2].max()} ns")
