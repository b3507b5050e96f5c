"""Phase-1 (k_b_refactor warp tasks) per-warp cycle accounting under KKT_TRACE=1: where the
warps of the batched replay spend their cycles (batch.cu PROF_MARK)."""
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
nst = max(int(f._so_ptr[-1]), 4 * f.n)
stp = np.zeros(nst, dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace_steps(dev.h, stp.ctypes.data_as(C.c_void_p)))
nw = 740 * 4
c = stp[:8 * nw].reshape(nw, 8).astype(np.float64)
names = ["dispatch+meta", "A scatter", "staging issue", "wait staged", "replay", "finalize", "tasks", "staged vals"]
tot = c[:, :6].sum()
for i in range(6):
    print(f"{names[i]:14s} {100 * c[:, i].sum() / tot:5.1f}%  ({c[:, i].sum() / nw / 1.9e3:8.1f} us per warp)")
print(f"tasks per warp {c[:, 6].mean():.1f}; warps {nw}")
ref = np.zeros(2 * f.n, dtype=np.uint64)
tri = np.zeros(2 * f.n, dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace(dev.h, ref.ctypes.data_as(C.c_void_p), tri.ctypes.data_as(C.c_void_p)))
ntask = int(np.count_nonzero(ref[1::2]))
end = ref[1::2][:ntask].astype(np.int64)
st = stp[100000:100000 + 2 * ntask:2].astype(np.int64)
col = stp[100001:100001 + 2 * ntask:2].astype(np.int64)
t0 = st[st > 0].min()
st, end = (st - t0) / 1e3, (end - t0) / 1e3
so, sod = f._so_ptr, f._so_data
n = f.n
lev = np.zeros(n, int)
for j in range(n):
    ks = sod[so[j]:so[j + 1]]
    if len(ks):
        lev[j] = lev[ks].max() + 1
L = lev[col]
print(f"phase-1 tasks {ntask}: span {end.max():.0f} us, levels {L.min()}..{L.max()}")
# per level: first start, last end, tasks
for l in list(range(L.min(), L.max() + 1))[:: max(1, (L.max() - L.min()) // 30)]:
    m = L == l
    if m.any():
        print(f"  level {l:4d}: {m.sum():6d} tasks  start {st[m].min():8.1f}..{st[m].max():8.1f}  end {end[m].min():8.1f}..{end[m].max():8.1f} us")
dur = end - st
print(f"task duration us: p10 {np.percentile(dur, 10):.1f} p50 {np.percentile(dur, 50):.1f} p90 {np.percentile(dur, 90):.1f}")
