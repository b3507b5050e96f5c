"""Chain-task grid phases (single system, KKT_TRACE=1): per-row publish times -> intra-chain
link time, chain start after its last external dependency, one-row hop, and the critical
path split into those classes.  usage: trace_chain.py CONFIG"""
import ctypes as C
import os
import sys

os.environ["KKT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_rhs, system_values

cfg = sys.argv[1] if len(sys.argv) > 1 else "activsg10k"
pat = build_pattern(ACOPF_CONFIGS[cfg], 0)
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
dev = f.device(restart_m=10)
rhs = system_rhs(pat, 1, 0)
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
Lc = sp.csc_matrix((np.ones(len(f._Li)), f._Li, f._Lp), shape=(n, n)).tocsr()
Uc = sp.csc_matrix((np.ones(len(f._Ui)), f._Ui, f._Up), shape=(n, n)).tocsr()
for name, off, p, M, up in (("L", 0, pL, Lc, False), ("U", n, pU, Uc, True)):
    tt = t[off:off + p]
    rp, ci = M.indptr, M.indices
    traced = tt > 0
    order = range(p - 1, -1, -1) if up else range(p)
    head = np.full(p, -1)
    ln = np.zeros(p, int)
    for r in order:
        if not traced[r]:
            continue
        prev = r + 1 if up else r - 1
        cols = ci[rp[r]:rp[r + 1]]
        cols = cols[cols < p]
        link = 0 <= prev < p and traced[prev] and len(cols) and (cols.min() if up else cols.max()) == prev \
            and ln[head[prev]] < 32
        head[r] = head[prev] if link else r
        ln[head[r]] += 1
    t0 = tt[traced].min()
    last = np.zeros(p, np.int64)
    lastc = np.full(p, -1)
    intra, start, single = [], [], []
    for r in order:
        if not traced[r]:
            continue
        cols = ci[rp[r]:rp[r + 1]]
        cols = cols[(cols < p)]
        cols = cols[traced[cols]]
        ext = cols[head[cols] != head[r]] if len(cols) else cols
        if len(ext):
            k = ext[np.argmax(tt[ext])]
            last[r], lastc[r] = tt[k], k
    for h in np.unique(head[traced]):
        m = ln[h]
        rows = [h - i if up else h + i for i in range(m)]
        if m == 1:
            if lastc[h] >= 0:
                single.append(tt[h] - last[h])
            continue
        ext_last = max(last[r] for r in rows)
        start.append(tt[rows[0]] - ext_last)
        intra += list(np.diff(tt[rows]))
    pr = lambda a: f"median {np.median(a):.0f} p90 {np.percentile(a, 90):.0f} ns (n={len(a)})" if len(a) else "-"
    print(f"{name} grid: span {(tt[traced].max() - t0) / 1e3:.1f} us; intra-chain link {pr(intra)}; "
          f"chain start after last external {pr(start)}; one-row hop {pr(single)}")
    # critical path back from the last row
    r = int(np.argmax(np.where(traced, tt, 0)))
    cls = {"intra": 0, "chain-start": 0, "one-row": 0}
    cnt = {"intra": 0, "chain-start": 0, "one-row": 0}
    while True:
        h = head[r]
        pos = (h - r) if up else (r - h)
        if pos > 0:
            prv = r + 1 if up else r - 1
            cls["intra"] += tt[r] - tt[prv]; cnt["intra"] += 1
            r = prv
            continue
        rows = [h - i if up else h + i for i in range(ln[h])]
        cand = [(last[q], lastc[q]) for q in rows if lastc[q] >= 0]
        if not cand:
            break
        lt, k = max(cand)
        key = "chain-start" if ln[h] > 1 else "one-row"
        cls[key] += tt[r] - lt; cnt[key] += 1
        r = int(k)
    print("   critical path: " + ", ".join(f"{k} {cnt[k]} x -> {v / 1e3:.1f} us" for k, v in cls.items()))
