"""Analyse gpurun_out/task_cycles.npy (KKT_TRACE=1 probe_kernels.py CFG 64 1 --tasks): per
batched-refactor task cycles grouped by the column's pattern size and systems per task."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_values

NB, XB, (LO, MID, HI) = 64, 768, (64, 256, 1024)
pat = build_pattern(ACOPF_CONFIGS["activsg10k"], 0)
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
n = f.n
Lc, Uc = np.diff(f._Lp), np.diff(f._Up)
npat = Lc + Uc + 1
so, sod = f._so_ptr, f._so_data
lev = np.zeros(n, int)
for j in range(n):
    ks = sod[so[j]:so[j + 1]]
    if len(ks):
        lev[j] = lev[ks].max() + 1
order = np.argsort(lev, kind="stable")
cnt = np.bincount(lev)
start = 0
l = 0
while l < 2 and cnt[l] >= 2048 and npat[lev == l].max() <= 64:
    start += cnt[l]
    l += 1
col_of = np.repeat(np.arange(n), np.diff(so))
pairs = np.bincount(col_of, weights=Lc[sod], minlength=n)
tasks = []
for c in order[start:]:
    S = 32
    while S > 1 and npat[c] * S > XB:
        S //= 2
    if pairs[c] > HI:
        S = 1
    elif pairs[c] > MID:
        S = min(S, 4)
    elif pairs[c] > LO:
        S = min(S, 8)
    tasks += [(c, S)] * (NB // S)
dur = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/task_cycles.npy")[:len(tasks)]
tc = np.array([t[0] for t in tasks])
ts = np.array([t[1] for t in tasks])
tot = dur.sum()
print(f"{len(tasks)} tasks, total {tot:.3e} warp-cycles")
for lo, hi in ((0, 8), (8, 16), (16, 32), (32, 64), (64, 128), (128, 256), (256, 10**9)):
    m = (npat[tc] > lo) & (npat[tc] <= hi)
    if m.any():
        print(f"np in ({lo},{hi}]: tasks {m.sum():7d} share {dur[m].sum() / tot:6.1%}  mean {dur[m].mean():9.0f} cyc  "
              f"S {np.bincount(ts[m]).nonzero()[0].tolist()}  pairs/task {(pairs[tc][m] * ts[m] / 1).mean():.0f}")
