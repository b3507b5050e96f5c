"""Timeline of one refactorization (KKT_TRACE=1): per-level dispatch/finish statistics."""
import ctypes as C
import os
import sys

os.environ["KKT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import make_sequence

seq = make_sequence(sys.argv[1] if len(sys.argv) > 1 else "activsg10k", seed=0, length=20)
f, _ = factorize(to_general(seq.matrix(0)))
dev = f.device()
n = f.n
with torch.cuda.stream(dev.stream):
    vals = torch.from_numpy(seq.values(19)).cuda()
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
for _ in range(2):
    dev.refactor_device(vals, nat.LAYOUT_SYMMETRIC_LOWER)
    dev.solve_device(b, x)
dev.sync()
tr = np.zeros(2 * n, dtype=np.uint64)
ts = np.zeros(2 * n, dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace(dev.h, tr.ctypes.data_as(C.c_void_p), ts.ctypes.data_as(C.c_void_p)))
st, en = tr[0::2].astype(np.int64), tr[1::2].astype(np.int64)
t0 = st.min()
st, en = (st - t0) / 1e3, (en - t0) / 1e3  # us
sop, sod = f._so_ptr, f._so_data
lev = np.zeros(n, np.int64)
for j in range(n):
    ks = sod[sop[j]:sop[j + 1]]
    if ks.size:
        lev[j] = lev[ks].max() + 1
print(f"refactor span {en.max():.1f} us")
for a, bnd in [(0, 1), (1, 2), (2, 5), (5, 20), (20, 50), (50, 100), (100, 200), (200, 300),
               (300, 400), (400, 600)]:
    m = (lev >= a) & (lev < bnd)
    if not m.any():
        continue
    dur = en[m] - st[m]
    print(f"levels [{a},{bnd}): cols {m.sum():7d} dispatch {st[m].min():8.1f}..{st[m].max():8.1f} "
          f"finish {en[m].min():8.1f}..{en[m].max():8.1f} us; per-col dur med {np.median(dur):7.2f} "
          f"max {dur.max():8.2f}")
# hop decomposition on the deep chain: F(k*) -> step k* applied in column j -> F(j)
steps = np.zeros(sod.size, dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace_steps(dev.h, steps.ctypes.data_as(C.c_void_p)))
late = (steps & np.uint64(1)).astype(bool)
stt = ((steps & ~np.uint64(1)).astype(np.int64) - t0) / 1e3
deep = np.flatnonzero(lev >= 300)
det, fin, prev = [], [], []
for j in deep:
    a, b = sop[j], sop[j + 1]
    if b - a < 2:
        continue
    k = sod[b - 1]
    det.append(stt[b - 1] - en[k])
    fin.append(en[j] - stt[b - 1])
    prev.append(stt[b - 1] - stt[b - 2])
print(f"deep hop: F(k*)->applied median {np.median(det):.2f} us, applied->F(j) median {np.median(fin):.2f} us, "
      f"gap between last two steps median {np.median(prev):.2f} us; late-step fraction {late[sop[deep[0]]:].mean():.2f}")
# trisolve L/U grid rows
tl = ts[:n].astype(np.int64)
tu = ts[n:].astype(np.int64)
for name, t in (("L", tl), ("U", tu)):
    t = t[t > 0]
    if t.size:
        print(f"trisolve {name} grid rows published over {(t.max() - t.min()) / 1e3:.1f} us")
# trisolve L grid hop: publish(r) - publish(critical dep) for rows in the narrow levels
info = dev.info()
pL = info["pL"]
Lp_, Li_ = f._Lp, f._Li
rows_of = [[] for _ in range(n)]
levL = np.zeros(n, np.int64)
# CSR of L: row r's columns
order = np.argsort(Li_, kind="stable")
cols = np.repeat(np.arange(n), np.diff(Lp_))[order]
rr = Li_[order]
rptr = np.zeros(n + 1, np.int64)
np.cumsum(np.bincount(rr, minlength=n), out=rptr[1:])
for r in range(n):
    cs = cols[rptr[r]:rptr[r + 1]]
    if cs.size:
        levL[r] = levL[cs].max() + 1
tl = ts[:n].astype(np.int64)
hops = []
for r in range(pL):
    cs = cols[rptr[r]:rptr[r + 1]]
    if cs.size == 0 or levL[r] < 50:
        continue
    c = cs[np.flatnonzero(levL[cs] == levL[cs].max())[-1]]
    if tl[r] and tl[c]:
        hops.append((tl[r] - tl[c]) / 1e3)
if hops:
    hops = np.array(hops)
    print(f"L grid hop (levels>=50): median {np.median(hops):.2f} us, p90 {np.percentile(hops, 90):.2f} us, n={hops.size}")
# deep columns: time from the last dependency finishing to the column finishing, and how many
# of the column's steps come after that dependency in so order (work left once it arrives)
after, nafter, cnt_after = [], [], []
for j in deep:
    a, b = sop[j], sop[j + 1]
    if b == a:
        continue
    ks = sod[a:b]
    crit = int(np.argmax(en[ks]))
    after.append(en[j] - en[ks[crit]])
    nafter.append(b - a - crit)
    cnt_after.append(int(sum(Lp_[k + 1] - Lp_[k] for k in ks[crit:])) if 'Lp_' in dir() else 0)
if after:
    after = np.array(after)
    print(f"deep columns: last dependency -> finish median {np.median(after):.2f} us, p90 "
          f"{np.percentile(after, 90):.2f}; steps at/after it median {np.median(nafter):.0f}, p90 "
          f"{np.percentile(nafter, 90):.0f}; L entries of those steps median {np.median(cnt_after):.0f}")
# per-step timing inside the deep columns: a step whose column k finished before the previous
# step was applied is pure work (time = apply(t) - apply(t-1)); otherwise it waited for k
work, waitd, nst = [], [], []
for j in deep:
    a, b = sop[j], sop[j + 1]
    nst.append(b - a)
    for t in range(a + 1, b):
        k = sod[t]
        d = stt[t] - stt[t - 1]
        if en[k] < stt[t - 1]:
            work.append(d)
        else:
            waitd.append(stt[t] - en[k])
work, waitd = np.array(work), np.array(waitd)
print(f"deep steps: {np.median(nst):.0f} per column (max {max(nst)}); ready steps {work.size}: median "
      f"{np.median(work):.3f} us, sum per column {work.sum() / len(deep):.1f} us; waiting steps "
      f"{waitd.size}: apply-after-F median {np.median(waitd):.2f} us")
