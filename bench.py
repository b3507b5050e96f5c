"""Benchmark: ms per KKT system (refactor + solve + FGMRES-IR) at ACTIVSg10k on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config activsg10k] [--tol barrier|fixed]

A "step" = one system of the ACOPF-shaped, ill-conditioned sequence:
refactorize on the frozen host analysis -> lu_solve -> refine_fgmres with the barrier-tied
tolerance delta(mu) (harness._run_direct_family, harness.py:223-245).  System 0 is
analysed once on the host (reported separately, like the reference's first factorize);
steps cycle over systems 1..M-1.

value  : device-resident inputs (values + rhs already in HBM), CUDA-event time per step,
         L2 flushed between steps (256 MiB write, excluded from the timing).
e2e    : the same step through the C ABI with HOST buffers (values+rhs H2D, x D2H inside).
roofline: the dominant kernel family, algorithmic bytes per launch / event time.
cpu_baseline: the CPU oracle port (oracle/kkt_oracle.c) on a bounded sample on this host.
--impl reference: the reference arm = the oracle port on all host threads (the reference is
         pure Python/numpy and cannot be installed on the box; DESIGN.md §Reference arm).
Multi-GPU (torchrun): independent systems sharded across ranks, no collective on the data
path; value = max-over-ranks time / systems processed by all ranks ("weak").
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per KKT system (refactor+solve+IR) at ACTIVSg10k; HBM GB/s vs peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=19)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="activsg10k")
    ap.add_argument("--systems", type=int, default=20)
    ap.add_argument("--tol", default="barrier", choices=["barrier", "fixed"])
    ap.add_argument("--delta", type=float, default=1e-10)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=5)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def make_problem(config: str, systems: int):
    from paper_2401_13926_b200.acopf import make_sequence
    t = time.perf_counter()
    seq = make_sequence(config, seed=0, length=systems)
    gen_s = time.perf_counter() - t
    vals = [seq.values(k) for k in range(systems)]
    rhs = [seq.rhs(k) for k in range(systems)]
    mus = [seq.mu(k) for k in range(systems)]
    return seq, vals, rhs, mus, gen_s


def policy_of(args):
    from paper_2401_13926_b200.refine import BarrierTiedTolerance, FixedTolerance
    return BarrierTiedTolerance() if args.tol == "barrier" else FixedTolerance(args.delta)


def oracle_factors(f, K0):
    from oracle import oracle
    from paper_2401_13926_b200.sparse import expand_pattern
    ex = expand_pattern(K0)
    arrays = dict(row_perm=f.row_perm.perm, col_perm=f.col_perm.perm, Lp=f._Lp, Li=f._Li,
                  Lx=f._Lx, Up=f._Up, Ui=f._Ui, Ux=f._Ux, Udiag=f._Udiag, so_ptr=f._so_ptr,
                  so_data=f._so_data, ap_ptr=f._ap_ptr, a_src=f._a_src, a_tgt=f._a_tgt)
    return oracle.OracleFactors(arrays, ex.general.row_ptr), ex


def cpu_port_time(f, seq, vals, rhs, mus, policy, budget_s: float, threads: int = 1,
                  start: int = 1):
    """Oracle port: per-system refactorize + lu_solve + refine_fgmres on host cores."""
    from concurrent.futures import ThreadPoolExecutor
    K0 = seq.matrix(0)
    M = len(vals)
    done = []
    t_all = time.perf_counter()
    lock = threading.Lock()

    def worker(wid):
        of, ex = oracle_factors(f, K0)
        i = start + wid
        while time.perf_counter() - t_all < budget_s or not done:
            k = 1 + (i - 1) % (M - 1)
            t0 = time.perf_counter()
            of.refactorize(vals[k][ex.src])
            x0 = of.lu_solve(rhs[k])
            of.refine_fgmres(K0.row_ptr, K0.col_idx, vals[k], rhs[k], x0, policy(mus[k]))
            dt = time.perf_counter() - t0
            with lock:
                done.append(dt)
            i += threads

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(worker, range(threads)))
    wall = time.perf_counter() - t_all
    return wall, len(done), float(np.mean(done))


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2401_13926_b200 import factorize, to_general
    seq, vals, rhs, mus, _ = make_problem(args.config, args.systems)
    f, _ = factorize(to_general(seq.matrix(0)))
    threads = os.cpu_count() or 1
    policy = policy_of(args)
    budget = max(2.0, args.cpu_seconds / max(1, args.steps + args.warmup) * args.steps)
    cpu_port_time(f, seq, vals, rhs, mus, policy, 0.5, threads)  # warm-up
    wall, n_sys, mean_one = cpu_port_time(f, seq, vals, rhs, mus, policy, budget, threads)
    value = wall * 1e3 / n_sys
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ms/system",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} ACOPF-shaped KKT sequence, refactor+solve+IR",
                   "N": seq.pattern.N, "nnz_lower": seq.pattern.K.nnz},
        "cpu_baseline": {"value": value, "unit": "ms/system", "cores": threads, "kind": "port",
                         "sample": f"{n_sys} systems of the sequence in {wall:.1f}s "
                                   f"({threads} threads, one system per thread)"},
        "e2e": {"value": value, "unit": "ms/system", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200 import factorize, to_general

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    seq, vals, rhs, mus, gen_s = make_problem(args.config, args.systems)
    K0 = seq.matrix(0)
    M = args.systems
    t0 = time.perf_counter()
    f, _ = factorize(to_general(K0))
    analyze_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev = f.device(restart_m=10)
    create_s = time.perf_counter() - t0
    if local != 0 and dev.device.index != local:
        raise RuntimeError("device mismatch")
    policy = policy_of(args)
    N = seq.pattern.N
    nnz_lower = seq.pattern.K.nnz
    st = f.stats
    stream = dev.stream
    lib = dev.lib

    # ---- device-resident inputs ----
    with torch.cuda.stream(stream):
        dvals = torch.from_numpy(np.stack(vals)).to(dev.device)
        drhs = torch.from_numpy(np.stack(rhs)).to(dev.device)
        dx = torch.empty(N, dtype=torch.float64, device=dev.device)
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev.device)
    stream.synchronize()

    def flush_l2():
        with torch.cuda.stream(stream):
            flush.fill_(1.0)

    # systems for this rank: shard the sequence round-robin (independent units)
    def system_of(step):
        return 1 + (rank + world * step) % (M - 1)

    def run_step(k, on_device=True, hv=None, hr=None, hx=None):
        d = policy(mus[k])
        if on_device:
            return dev.step(dvals[k], nat.LAYOUT_SYMMETRIC_LOWER, drhs[k], dx, True, 10, 10, d)
        return dev.step(hv, nat.LAYOUT_SYMMETRIC_LOWER, hr, hx, False, 10, 10, d)

    for w in range(args.warmup):
        run_step(system_of(w))
    launches0 = dev.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    iters = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for s in range(args.steps):
            flush_l2()
            ev[s][0].record(stream)
            rep = run_step(system_of(args.warmup + s))
            ev[s][1].record(stream)
            iters.append(rep.iterations)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    launches = dev.launch_count() - launches0
    total_ms = float(np.sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], device=dev.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = total_ms / (args.steps * world)

    # ---- e2e through the C ABI with host (pinned) buffers ----
    hv = [torch.from_numpy(v).pin_memory().numpy() for v in vals]
    hr = [torch.from_numpy(r).pin_memory().numpy() for r in rhs]
    hx = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
    for w in range(2):
        k = system_of(w)
        run_step(k, False, hv[k], hr[k], hx)
    e2e_ms = []
    for s in range(args.steps):
        k = system_of(args.warmup + s)
        flush_l2()
        stream.synchronize()
        t0 = time.perf_counter()
        run_step(k, False, hv[k], hr[k], hx)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_total = float(np.sum(e2e_ms))
    if dist:
        t = torch.tensor([e2e_total], device=dev.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = e2e_total / (args.steps * world)

    # ---- per-kernel roofline (trisolve pair, SpMV, refactor), flushed L2 ----
    nL, nU = st["nnz_L"], st["nnz_U"]
    nnz_g = st["nnz_general"]
    pairs = st["update_pairs"]
    bytes_tri = 12 * (nL + nU) + 8 * N + 8 * (N + 1) * 2 + N * 12 + 2 * 8 * N + N * 12
    bytes_spmv = 12 * nnz_g + 4 * (N + 1) + 4 * N + 8 * N + 8 * N
    bytes_ref = (8 * nnz_lower + 8 * nnz_g + 4 * (nL + nU) + 4 * nU + 8 * (nL + nU + N)
                 + 2 * pairs + 8 * (nL + nU))
    with torch.cuda.stream(stream):
        xb = torch.randn(N, dtype=torch.float64, device=dev.device)
        yb = torch.empty(N, dtype=torch.float64, device=dev.device)

    def timed(fn, reps):
        out = []
        for _ in range(reps):
            flush_l2()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            out.append(a.elapsed_time(b))
        return float(np.median(out))

    t_tri = timed(lambda: dev.solve_device(xb, yb), args.kernel_reps)
    t_spmv = timed(lambda: dev.spmv_device(xb, yb), args.kernel_reps)
    t_ref = timed(lambda: dev.refactor_device(dvals[M - 1], nat.LAYOUT_SYMMETRIC_LOWER),
                  args.kernel_reps)
    peak, peak_kind = peaks()
    kern = {
        "trisolve_pair": {"ms": t_tri, "bytes": bytes_tri, "GBs": bytes_tri / t_tri / 1e6},
        "spmv": {"ms": t_spmv, "bytes": bytes_spmv, "GBs": bytes_spmv / t_spmv / 1e6},
        "refactor": {"ms": t_ref, "bytes": bytes_ref, "GBs": bytes_ref / t_ref / 1e6,
                     "flops": st["refactor_flops"],
                     "GFLOPs": st["refactor_flops"] / t_ref / 1e6},
    }
    mean_iters = float(np.mean(iters)) if iters else 0.0
    share = {"trisolve_pair": t_tri * (1 + mean_iters), "refactor": t_ref,
             "spmv": t_spmv * (mean_iters + 3)}
    dom = max(share, key=share.get)
    kd = kern[dom]

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        wall, n_sys, mean_one = cpu_port_time(f, seq, vals, rhs, mus, policy,
                                              args.cpu_seconds, threads=1)
        cpu = {"value": mean_one * 1e3, "unit": "ms/system", "cores": 1, "kind": "port",
               "sample": f"{n_sys} systems (refactorize+lu_solve+refine_fgmres) of the same "
                         f"sequence, single thread, {wall:.1f}s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "ms/system", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {
                "workload": f"{args.config}-shaped ill-conditioned KKT sequence: per system "
                            "refactor + lu_solve + FGMRES(10)-IR (CGS2), barrier-tied tol"
                            if args.tol == "barrier" else f"fixed delta={args.delta}",
                "N": N, "nnz_lower": nnz_lower, "nnz_general": nnz_g, "nnz_L": nL, "nnz_U": nU,
                "refactor_flops": st["refactor_flops"],
                "levels_refactor_L_U": [st["refactor_levels"], st["L_levels"], st["U_levels"]],
                "offdiag_pivots": st["offdiag_pivots"], "systems": M,
                "tolerance": "delta(mu)=clamp(1e-2*mu,1e-10,1e-8)" if args.tol == "barrier"
                else f"{args.delta}",
                "mean_ir_iterations": mean_iters,
                "l2": "flushed between steps (256 MiB write, excluded from timing)",
                "analyze_s": analyze_s, "device_create_s": create_s, "generate_s": gen_s,
                "parallelism": f"replicas/shards x{world}",
                "step_ms": [round(x, 4) for x in step_ms],
                "schedule": dev.info(),
            },
            "e2e": {"value": e2e_value, "unit": "ms/system",
                    "h2d_bytes_per_step": 8 * (nnz_lower + N), "d2h_bytes_per_step": 8 * N},
            "roofline": {"kernel": dom, "bound": "hbm", "achieved": kd["GBs"], "peak": peak,
                         "unit": "GB/s", "frac": kd["GBs"] / peak, "traffic": None,
                         "peak_kind": peak_kind,
                         "note": "single-system trisolve/refactor are DAG-latency bound "
                                 "(levels x hop latency); see DESIGN.md"},
            "kernels": kern,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
