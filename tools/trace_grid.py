"""Grid-phase trisolve timeline (KKT_TRACE=1): per-row publish times of system 0 ->
kernel span, level-front progression and the hop latency after the last dependency.
usage: trace_grid.py CONFIG B"""
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

cfg, B = sys.argv[1], int(sys.argv[2])
pat = build_pattern(ACOPF_CONFIGS[cfg], 0)
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
dev = DeviceSystem(f, batch=B)
rhs = np.stack([system_rhs(pat, 1 + q % 19, q // 19) for q in range(B)]) if B > 1 else system_rhs(pat, 1, 0)
with torch.cuda.stream(dev.stream):
    tr = torch.from_numpy(rhs).to(dev.device)
    tx = torch.empty_like(tr)
for _ in range(3):
    dev.solve_device(tr, tx)
dev.sync()
n = f.n
info = dev.info()
pL, pU = info["pL"], info["pU"]
ref = np.zeros(2 * n, dtype=np.uint64)
tri = np.zeros(2 * n, dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace(dev.h, ref.ctypes.data_as(C.c_void_p), tri.ctypes.data_as(C.c_void_p)))
t = tri.astype(np.int64)
steps = np.zeros(max(int(f._so_data.size), 4 * n), dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace_steps(dev.h, steps.ctypes.data_as(C.c_void_p)))
stt = steps.astype(np.int64)
# dependencies: L row r <- columns of L(r, :) ; U row r <- columns of U(r, :)
Lp, Li = f._Lp, f._Li
Up, Ui = f._Up, f._Ui
for name, off, p, colp, rowi in (("L", 0, pL, Lp, Li), ("U", n, pU, Up, Ui)):
    tt = t[off:off + p]
    if not (tt > 0).all():
        print(name, "incomplete trace", (tt > 0).sum(), p)
        continue
    t0 = tt.min()
    # last dependency time per row (deps in the grid part only)
    cols = np.repeat(np.arange(n), np.diff(colp))
    m = (rowi < p) & (cols < p)
    last = np.zeros(p, dtype=np.int64)
    np.maximum.at(last, rowi[m], tt[cols[m]])
    has = np.zeros(p, bool)
    has[rowi[m]] = True
    hop = (tt - last)[has]
    span = tt.max() - t0
    q = np.percentile(tt - t0, [10, 50, 90, 99, 100])
    print(f"{name} grid (B={B}): span {span / 1e3:.1f} us; publish-time pct 10/50/90/99/100: "
          + " ".join(f"{v / 1e3:.0f}" for v in q) + " us; hop after last dep: median "
          f"{np.median(hop):.0f} ns, p90 {np.percentile(hop, 90):.0f} ns, mean {hop.mean():.0f} ns")
    # critical path: follow the latest dependency backwards from the last row
    r = int(np.argmax(tt))
    path = [r]
    depmap = {}
    while True:
        ds = [c for c in (cols[m][rowi[m] == r])]
        if not ds:
            break
        r = max(ds, key=lambda c: tt[c])
        path.append(r)
        if len(path) > 5000:
            break
    hops = -np.diff(tt[path])
    print(f"   critical chain {len(path)} rows, mean hop {hops.mean():.0f} ns, chain start at "
          f"{(tt[path[-1]] - t0) / 1e3:.1f} us")
    if B > 1:
        st0 = stt[2 * off // 1 + 0: 2 * (off + p): 2] if False else stt[2 * off:2 * (off + p):2]
        stc = stt[2 * off + 1:2 * (off + p):2]
        ok = (st0 > 0) & has
        if ok.any():
            q = (st0 - last)[ok]   # start after the last dependency was published (queueing)
            w = (stc - st0)[ok]    # critical-dependency wait
            k = (tt - stc)[ok]     # work after the dependency: reloads, sum, publish
            pth = [r for r in path if ok[r]]
            print(f"   rows: start-after-deps median {np.median(q):.0f} ns (p90 {np.percentile(q, 90):.0f}), "
                  f"crit wait median {np.median(w):.0f}, work median {np.median(k):.0f} ns")
            if pth:
                pq = (st0 - last)[pth]; pw = (stc - st0)[pth]; pk = (tt - stc)[pth]
                print(f"   on the critical chain: start-after-deps mean {pq.mean():.0f} ns, crit wait "
                      f"{pw.mean():.0f}, work {pk.mean():.0f} ns")
