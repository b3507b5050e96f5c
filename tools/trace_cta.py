"""Phase-2 (k_b_refactor_cta) task trace (KKT_TRACE=1): start/end/column of every
(column, system group) task -> where the wide-column replay spends its time: dispatch lag,
waiting on dependency columns, or own steps after the last dependency landed."""
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
SC = int(os.environ.get("KKT_B_CT_SC", "8"))
pat = build_pattern(ACOPF_CONFIGS["activsg10k"], 0)
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
dev = DeviceSystem(f, batch=B)
vals = np.stack([system_values(pat, 1 + q % 19, q // 19) for q in range(B)])
with torch.cuda.stream(dev.stream):
    tv = torch.from_numpy(vals).to(dev.device)
for _ in range(3):
    dev.refactor_device(tv, nat.LAYOUT_SYMMETRIC_LOWER)
dev.sync()
n = f.n
ref = np.zeros(2 * n, dtype=np.uint64)
tri = np.zeros(2 * n, dtype=np.uint64)
nat.check(dev.lib.kkt_dev_trace(dev.h, ref.ctypes.data_as(C.c_void_p), tri.ctypes.data_as(C.c_void_p)))
W = 8 if os.environ.get('KKT_B_CT_MODE') == '3' else 4
tr = tri.reshape(-1, W)
ntask = int(np.count_nonzero(tr[:, 0]))
st, en, col = tr[:ntask, 0].astype(np.int64), tr[:ntask, 1].astype(np.int64), tr[:ntask, 2].astype(np.int64)
ngrp = (B + 31) // 32 * 32 // SC
t0 = st.min()
st, en = st - t0, en - t0
grp = np.arange(ntask) % ngrp
end_of = {}
for t in range(ntask):
    end_of[(int(col[t]), int(grp[t]))] = en[t]
J2 = col.min()
so, sod = f._so_ptr, f._so_data
dep_end = np.zeros(ntask, np.int64)
nsteps = np.zeros(ntask, np.int64)
ndep = np.zeros(ntask, np.int64)
for t in range(ntask):
    j = int(col[t])
    ks = sod[so[j]:so[j + 1]]
    nsteps[t] = len(ks)
    ks = ks[ks >= J2]
    ndep[t] = len(ks)
    if len(ks):
        dep_end[t] = max(end_of[(int(k), int(grp[t]))] for k in ks)
dur = en - st
after = en - np.maximum(st, dep_end)
print(f"tasks {ntask}  makespan {en.max() / 1e3:.1f} us  sum dur {dur.sum() / 1e6:.1f} ms")
for name, a in (("duration", dur), ("after last dep", after), ("start lag behind dep", np.maximum(0, st - dep_end))):
    print(f"{name:22s} us: mean {a.mean() / 1e3:7.2f}  p50 {np.percentile(a, 50) / 1e3:7.2f}  "
          f"p90 {np.percentile(a, 90) / 1e3:7.2f}  max {a.max() / 1e3:7.2f}")
per = after / np.maximum(nsteps, 1)
print(f"ns per step after last dep: p50 {np.percentile(per, 50):.1f}  p90 {np.percentile(per, 90):.1f}")
# critical chain: walk back from the last task through the binding dependency
t = int(np.argmax(en))
chain = []
pos = {(int(col[i]), int(grp[i])): i for i in range(ntask)}
while True:
    chain.append(t)
    j = int(col[t])
    ks = sod[so[j]:so[j + 1]]
    ks = ks[ks >= J2]
    if not len(ks) or dep_end[t] <= st[t]:
        break
    t = max((pos[(int(k), int(grp[t]))] for k in ks), key=lambda i: en[i])
print(f"critical chain: {len(chain)} tasks; first starts {st[chain[-1]] / 1e3:.1f} us")
gap = [(en[a] - en[b]) for a, b in zip(chain[:-1], chain[1:])]
print(f"  per link (end-to-end) us: mean {np.mean(gap) / 1e3:.2f}  p50 {np.median(gap) / 1e3:.2f}; "
      f"steps per link mean {np.mean([nsteps[c] for c in chain]):.0f}")
for c in chain[:8]:
    print(f"   col {col[c]} grp {grp[c]} st {st[c] / 1e3:.1f} dep {dep_end[c] / 1e3:.1f} en {en[c] / 1e3:.1f} steps {nsteps[c]} ndep {ndep[c]}")

if W == 8:
    ev = tr[:ntask, 3:7].astype(np.int64) - t0
    print("chain link anatomy (us after the binding dependency's end):")
    for c in chain[:10]:
        de = dep_end[c]
        f = lambda v: f"{(v - de) / 1e3:6.2f}" if v > 0 else "   -  "
        print(f"   col {col[c]}: flag seen {f(ev[c, 0])} last chunk {f(ev[c, 1])} steps done {f(ev[c, 2])} "
              f"fenced {f(ev[c, 3])} end {f(en[c])}")
