"""Batched refactor timeline (KKT_TRACE=1): end time of every k_b_refactor task vs its column
position -> when the light part and the heavy separator tail finish."""
import ctypes as C
import os
import sys

os.environ["KKT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_values
from paper_2401_13926_b200.device import DeviceSystem

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pat = build_pattern(ACOPF_CONFIGS["activsg10k"], 0)
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
dev = DeviceSystem(f, batch=B)
vals = np.stack([system_values(pat, 1 + q % 19, q // 19) for q in range(B)])
with torch.cuda.stream(dev.stream):
    tv = torch.from_numpy(vals).to(dev.device)
for _ in range(2):
    dev.refactor_device(tv, nat.LAYOUT_SYMMETRIC_LOWER)
dev.sync()
n = f.n
ref = np.zeros(2 * n, dtype=np.uint64)
tri = np.zeros(2 * n, dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace(dev.h, ref.ctypes.data_as(C.c_void_p), tri.ctypes.data_as(C.c_void_p)))
ntask = int(np.count_nonzero(ref[1::2]))
end = ref[1::2][:ntask].astype(np.int64)
dur = ref[0::2][:ntask].astype(np.float64)
t0 = end.min()
# rebuild the task -> column map (default policy: S from the workspace, XB = 768)
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
start, l = 0, 0
while l < 2 and cnt[l] >= 2048 and npat[lev == l].max() <= 64:
    start += cnt[l]
    l += 1
cols = []
for c in order[start:]:
    S = 32
    while S > 1 and npat[c] * S > 768:
        S //= 2
    cols += [c] * (-(-B // 32) * 32 // S)
cols = np.array(cols[:ntask])
e = (end - t0) / 1e3
print(f"B={B}: {ntask} tasks, span {e.max():.0f} us")
for lo, hi in ((0, 16), (16, 64), (64, 128), (128, 256), (256, 10**6)):
    m = (npat[cols] > lo) & (npat[cols] <= hi)
    if m.any():
        print(f"  np ({lo},{hi}]: {m.sum():6d} tasks, end-time pct 10/50/90/100: "
              + " ".join(f"{v:.0f}" for v in np.percentile(e[m], [10, 50, 90, 100])) + " us;"
              f" busy {dur[m].sum() / 1.9e3 / e.max():.0f} warp-equivalents")
pos_cut = np.where(npat > 64)[0].min()
m = cols >= pos_cut
print(f"  columns >= {pos_cut} (tail): first end {e[m].min():.0f} us, last {e[m].max():.0f} us; "
      f"columns < {pos_cut}: last end {e[~m].max():.0f} us")
