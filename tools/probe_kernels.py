"""Per-phase probe of the batched handle: refactor / solve timings (CUDA events), optional
step.  Usage: probe_kernels.py CONFIG B [reps] [--step]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200 import factorize, to_general
from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_rhs, system_values
from paper_2401_13926_b200.device import DeviceSystem

cfg = sys.argv[1]
B = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg_name, _, frac = cfg.partition("/")  # CONFIG or CONFIG/imbalance_frac
pat = build_pattern(ACOPF_CONFIGS[cfg_name], 0, imbalance_frac=float(frac or 1.0))
f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
dev = DeviceSystem(f, batch=B)
ks = [1 + q % 19 for q in range(B)]
vals = np.stack([system_values(pat, k, q // 19) for q, k in enumerate(ks)])
rhs = np.stack([system_rhs(pat, k, q // 19) for q, k in enumerate(ks)])
s = dev.stream
with torch.cuda.stream(s):
    tv = torch.from_numpy(vals).to(dev.device)
    tr = torch.from_numpy(rhs).to(dev.device)
    tx = torch.empty_like(tr)
s.synchronize()


def timed(fn):
    ts = []
    for _ in range(reps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        e.record(s)
        e.synchronize()
        ts.append(a.elapsed_time(e))
    return min(ts)


tref = timed(lambda: dev.refactor_device(tv, nat.LAYOUT_SYMMETRIC_LOWER))
tsol = timed(lambda: dev.solve_device(tr, tx))
line = (f"{cfg} B={B} sched={os.environ.get('KKT_B_SCHED', '-')} refactor {tref:8.3f} ms "
        f"({tref / B * 1e3:7.1f} us/sys)  solve {tsol:7.3f} ms ({tsol / B * 1e3:7.1f} us/sys)")
if "--step" in sys.argv:
    its = []

    def step():
        reps_ = dev.step(tv, nat.LAYOUT_SYMMETRIC_LOWER, tr, tx, True, 10, 10, 1e-10)
        reps_ = reps_ if isinstance(reps_, list) else [reps_]
        its.append(max(r.iterations for r in reps_))

    tstep = timed(step)
    line += f"  step {tstep:8.3f} ms ({tstep / B * 1e3:7.1f} us/sys, max its {its[-1]})"
print(line, flush=True)
if os.environ.get("KKT_TRACE") and B > 1:
    import ctypes as C
    dev.refactor_device(tv, nat.LAYOUT_SYMMETRIC_LOWER)
    s.synchronize()
    n_so = int(f._so_data.size)
    buf = np.zeros(n_so, dtype=np.uint64)
    nat.check(dev.lib.kkt_dev_trace_steps(dev.h, buf.ctypes.data_as(C.c_void_p)))
    info = dev.info()
    nw = info["refactor_blocks"] * info["refactor_warps"]
    pr = buf[:8 * nw].reshape(nw, 8).astype(np.float64)
    tot = pr[:, :6].sum()
    names = ["dispatch+meta", "A scatter", "staging", "producer wait", "replay", "finalize"]
    print("k_b_refactor per-warp cycle shares: " + ", ".join(
        f"{nm} {pr[:, k].sum() / tot:.1%}" for k, nm in enumerate(names)) +
        f"; tasks {pr[:, 6].sum():.0f}, staged values {pr[:, 7].sum():.3e}, "
        f"mean warp cycles {pr[:, :6].sum(1).mean():.3e}", flush=True)
if os.environ.get("KKT_TRACE") and B > 1 and "--tasks" in sys.argv:
    # per-task cycles (k_b_refactor) by column pattern size
    ref = np.zeros(2 * f.n, dtype=np.uint64)
    tri = np.zeros(2 * f.n, dtype=np.uint64)
    nat.check(dev.lib.kkt_dev_trace(dev.h, ref.ctypes.data_as(C.c_void_p), tri.ctypes.data_as(C.c_void_p)))
    # rebuild the task table like build_batch_tasks (default thresholds)
    Lc, Uc = np.diff(f._Lp), np.diff(f._Up)
    npat = Lc + Uc + 1
    so = f._so_ptr
    cnt = Lc[f._so_data]
    pairs = np.add.reduceat(np.append(cnt, 0), so[:-1])[:f.n] * (np.diff(so) > 0)
    info = dev.info()
    print("task-cycle histogram needs the plan order; raw stats:", np.count_nonzero(ref),
          "tasks, cycles total %.3e" % ref.astype(float).sum(), flush=True)
    dur = ref.astype(float)
    np.save("gpurun_out/task_cycles.npy", dur)
