"""One bench step (B systems of value streams 0..B-1 at barrier step k, kkt_dev_step with the
barrier-tied delta), repeated: for ncu launch lists / --set full captures of an IR step.

    python tools/step_probe.py CONFIG B K [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2401_13926_b200._native as nat
from paper_2401_13926_b200.device import DeviceSystem

cfg, B, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
args = bench.parse(["--config", cfg, "--imbalance-frac", os.environ.get("IMBALANCE_FRAC", "1.0")])
pat, f, _, _ = bench.setup(args)
vals, rhs, mu = bench.make_batch(pat, list(range(B)), k)
delta = bench.policy_of(args)(mu)
dev = DeviceSystem(f, batch=B) if B > 1 else f.device(restart_m=10)
with torch.cuda.stream(dev.stream):
    tv = torch.from_numpy(vals if B > 1 else vals[0]).to(dev.device)
    tr = torch.from_numpy(rhs if B > 1 else rhs[0]).to(dev.device)
    tx = torch.empty_like(tr)
for _ in range(reps):
    reps_ = dev.step(tv, nat.LAYOUT_SYMMETRIC_LOWER, tr, tx, True, 10, 10, delta, stats=True)
    reps_ = reps_ if isinstance(reps_, list) else [reps_]
    print("iterations", sorted(r.iterations for r in reps_), "handed", sum(r.handed_off for r in reps_),
          flush=True)
