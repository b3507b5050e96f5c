"""Benchmark: ms per KKT system (refactor + solve + FGMRES-IR) at ACTIVSg10k on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--global-batch 64] [--scaling strong|weak] [--config activsg10k]

Workload (BASELINE.json configs[4] with configs[2] beside it): ACOPF-shaped,
ill-conditioned KKT systems of one sparsity pattern (N = 238,080, nnz_lower = 716,700).
System 0 is analysed once on the host (reported separately, like the reference's first
`factorize`).  Every other system goes through the reference's per-system loop
(harness._run_direct_family, harness.py:223-245): refactorize on the frozen analysis ->
lu_solve -> refine_fgmres (trigger, FGMRES(10)-IR, nsr/nrbe after), with the barrier-tied
tolerance delta(mu).

A step = the global batch of 64 independent systems (value streams q = 0..63 of the pattern:
contingencies / time periods) at ONE barrier step k, as a batched interior-point method
advances its scenarios in lockstep; step s uses k = 1 + (s mod 19), so 19 steps cover the
whole barrier sequence once (early: no IR; late: up to 23 FGMRES iterations).  On N GPUs the
global batch is split 64/N systems per GPU ("scaling": "strong", configs[4]); --scaling weak
gives every GPU its own 64 systems instead.  value = max-over-ranks device time / systems.

value   : device-resident inputs, CUDA-event time per step, L2 flushed between steps (256 MiB
          write, untimed).
e2e     : the same steps through the public API with HOST (pinned) buffers: values and rhs
          H2D and x D2H inside the timed region, overlapped with the neighbouring steps'
          compute (pipeline.BatchPipeline).
sequence: configs[2] — the 19 systems of ONE value stream in barrier order on a
          single-system handle: device latency per system, e2e (host values in, x out through
          kkt_dev_step) and the single-thread CPU port on the same 19 systems.
fixed_delta: the batched steps again with the reference's fixed delta = 1e-10.
roofline: dominant kernel family, algorithmic bytes per launch / event time, and
          the critical-path bound (DAG levels x the measured inter-SM hop latency).
cpu_baseline: the CPU oracle port (oracle/kkt_oracle.c), one thread, on a deterministic
          subset of the timed systems.
--impl reference: the reference arm — the oracle port on every host thread over EXACTLY the
          GPU arm's (barrier step, value stream) list (the reference itself is pure
          Python/numpy and cannot travel to the box; the port is pinned bitwise to it).
Every timed system's convergence and true residual are checked; a non-converged system makes
the run exit 1 after printing its line.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per KKT system (refactor+solve+IR) at ACTIVSg10k; HBM GB/s vs peak"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=19)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="activsg10k")
    ap.add_argument("--global-batch", type=int, default=64)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--systems", type=int, default=20)
    ap.add_argument("--tol", default="barrier", choices=["barrier", "fixed"])
    ap.add_argument("--delta", type=float, default=1e-10)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single", action="store_true")
    ap.add_argument("--no-fixed", action="store_true")
    ap.add_argument("--no-handoff", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=3)
    ap.add_argument("--imbalance-frac", type=float, default=1.0,
                    help="fraction of buses with an imbalance slack; < 1 gives the reference's "
                         "off-diagonal pivoting regime (acopf.build_pattern)")
    return ap.parse_args(argv)


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
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def policy_of(args, fixed: bool = False):
    from paper_2401_13926_b200.refine import BarrierTiedTolerance, FixedTolerance
    if fixed or args.tol == "fixed":
        return FixedTolerance(args.delta)
    return BarrierTiedTolerance()


def step_k(s: int, M: int) -> int:
    """barrier step of bench step s: 1, 2, ..., M-1, 1, ... (19 steps = the whole sequence)"""
    return 1 + s % (M - 1)


def rank_seed_base(rank: int) -> int:
    """weak scaling: value streams of rank r are 1000 r + q, q < B — ranks never share one"""
    return 1000 * rank


def shard(rank: int, world: int, global_batch: int, scaling: str) -> list:
    """The value streams (systems of a step) rank `rank` processes.  strong: the global batch
    split in contiguous equal shards; weak: every rank its own global_batch systems."""
    if scaling == "weak":
        return [rank_seed_base(rank) + q for q in range(global_batch)]
    if global_batch % world:
        raise SystemExit(f"--global-batch {global_batch} does not split over {world} GPUs")
    per = global_batch // world
    return list(range(rank * per, (rank + 1) * per))


def job_streams(world: int, global_batch: int, scaling: str) -> list:
    """Every value stream of a step over all ranks (the reference arm's list)."""
    return [q for r in range(world) for q in shard(r, world, global_batch, scaling)]


def reduce_max(value: float, dist, device) -> float:
    """max over ranks (the job's time is its slowest rank's)"""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(value: float, dist, device) -> float:
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def make_batch(pat, streams, k: int):
    """The systems (value streams `streams`) at barrier step k: values [B][nnz_lower], rhs
    [B][N], mu_k."""
    from paper_2401_13926_b200.acopf import MU_STEP, system_rhs, system_values
    vals = np.stack([system_values(pat, k, q) for q in streams])
    rhs = np.stack([system_rhs(pat, k, q) for q in streams])
    return vals, rhs, 10.0 ** (-MU_STEP * k)


def oracle_factors(f, K0):
    from oracle import oracle
    from paper_2401_13926_b200.sparse import expand_pattern
    ex = expand_pattern(K0)
    arrays = dict(row_perm=f.row_perm.perm, col_perm=f.col_perm.perm, Lp=f._Lp, Li=f._Li,
                  Lx=f._Lx, Up=f._Up, Ui=f._Ui, Ux=f._Ux, Udiag=f._Udiag, so_ptr=f._so_ptr,
                  so_data=f._so_data, ap_ptr=f._ap_ptr, a_src=f._a_src, a_tgt=f._a_tgt)
    return oracle.OracleFactors(arrays, ex.general.row_ptr), ex


class CpuPort:
    """The oracle port on `threads` host threads, one system per thread at a time (the
    reference processes a system single-threaded): refactorize + lu_solve + refine_fgmres.
    The per-thread factor objects and the pool are built once, outside any timed region."""

    def __init__(self, f, K0, threads: int):
        from concurrent.futures import ThreadPoolExecutor
        self.K0, self.threads = K0, threads
        self.of = [oracle_factors(f, K0) for _ in range(threads)]
        self.pool = ThreadPoolExecutor(threads)

    def run(self, systems, policy, budget_s: float | None = None, round_len: int | None = None):
        """`systems` = list of (values, rhs, mu).  With a budget, stops at the first round
        boundary (round_len systems) after it.  Returns (wall_s, systems done, per-system s)."""
        import queue
        work = queue.Queue()
        for i in range(len(systems)):
            work.put(i)
        done = []
        lock = threading.Lock()
        stop = threading.Event()
        K0 = self.K0
        t_all = time.perf_counter()

        def worker(w):
            of, ex = self.of[w]
            while not stop.is_set():
                try:
                    i = work.get_nowait()
                except queue.Empty:
                    return
                vals, rhs, mu = systems[i]
                t0 = time.perf_counter()
                of.refactorize(vals[ex.src])
                x0 = of.lu_solve(rhs)
                of.refine_fgmres(K0.row_ptr, K0.col_idx, vals, rhs, x0, policy(mu))
                dt = time.perf_counter() - t0
                with lock:
                    done.append(dt)
                    if (budget_s is not None and time.perf_counter() - t_all > budget_s
                            and round_len and len(done) % round_len == 0):
                        stop.set()

        list(self.pool.map(worker, range(self.threads)))
        return time.perf_counter() - t_all, len(done), done

    def close(self):
        self.pool.shutdown()


def cpu_port_run(f, K0, systems, policy, threads: int, **kw):
    port = CpuPort(f, K0, threads)
    try:
        return port.run(systems, policy, **kw)
    finally:
        port.close()


def setup(args):
    from paper_2401_13926_b200 import factorize, to_general
    from paper_2401_13926_b200.acopf import ACOPF_CONFIGS, build_pattern, system_values
    t0 = time.perf_counter()
    pat = build_pattern(ACOPF_CONFIGS[args.config], 0, imbalance_frac=args.imbalance_frac)
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    f, _ = factorize(to_general(pat.K.with_values(system_values(pat, 0, 0))))
    return pat, f, gen_s, time.perf_counter() - t0


def gen_parallel(pat, items, threads: int):
    """system values / rhs for [(k, q)] on host threads (numpy releases the GIL)"""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2401_13926_b200.acopf import MU_STEP, system_rhs, system_values

    def one(kq):
        k, q = kq
        return system_values(pat, k, q), system_rhs(pat, k, q), 10.0 ** (-MU_STEP * k)

    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(one, items))


def workload_desc(args, world):
    per = args.global_batch // world if args.scaling == "strong" else args.global_batch
    return (f"{args.config}-shaped ill-conditioned KKT systems: per step a global batch of "
            f"{args.global_batch if args.scaling == 'strong' else args.global_batch * world} "
            f"independent same-pattern systems (value streams) at one barrier step, {per} per "
            f"GPU, refactor + lu_solve + refine_fgmres (FGMRES(10)-IR, CGS2) each; steps walk "
            f"barrier steps 1..{args.systems - 1}")


def run_reference(args, rank, world):
    """Reference arm: the oracle port on all host threads over exactly the GPU arm's systems."""
    if rank != 0:
        return
    world = max(world, args.gpus)
    pat, f, _, _ = setup(args)
    M = args.systems
    ks = [step_k(s, M) for s in range(args.steps)]
    streams = job_streams(world, args.global_batch, args.scaling)
    if len(streams) > 64:  # weak scaling at N > 1: a bounded sample of each step's systems
        streams = streams[:64]
    threads = os.cpu_count() or 1
    policy = policy_of(args)
    port = CpuPort(f, pat.K, threads)
    port.run(gen_parallel(pat, [(step_k(0, M), q) for q in streams[:threads]], threads), policy)
    wall = 0.0
    n_sys = 0
    step_ms = []
    for k in ks:
        systems = gen_parallel(pat, [(k, q) for q in streams], threads)
        w, n, _ = port.run(systems, policy)
        wall += w
        n_sys += n
        step_ms.append(round(w * 1e3, 2))
    value = wall * 1e3 / n_sys
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ms/system",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall * 1e3 / len(ks), "higher_is_better": False,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(args, world), "barrier_steps": ks,
                   "value_streams": [streams[0], streams[-1]], "systems_timed": n_sys,
                   "N": pat.N, "nnz_lower": pat.K.nnz, "global_batch": args.global_batch,
                   "step_ms": step_ms},
        "cpu_baseline": {"value": value, "unit": "ms/system", "cores": threads, "kind": "port",
                         "sample": f"all {n_sys} systems of the GPU arm's {len(ks)} steps "
                                   f"(value streams {streams[0]}..{streams[-1]} at barrier "
                                   f"steps {ks[0]}..{max(ks)}), {threads} threads, one system "
                                   "per thread; oracle/kkt_oracle.c"},
        "e2e": {"value": value, "unit": "ms/system", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    port.close()
    print(json.dumps(line), flush=True)


def spawn(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch as N ranks (one process per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def rr_of(rep) -> float:
    """true ||r - K x||_2 / ||r||_2 of the returned x (the harness's rr, harness.py:259-260)"""
    st = rep.stats_after if rep.triggered else rep.stats_before
    return st[0] / st[4] if st[4] > 0 else 0.0


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn(args))

    import torch
    import paper_2401_13926_b200._native as nat
    from paper_2401_13926_b200.device import DeviceSystem
    from paper_2401_13926_b200.pipeline import BatchPipeline

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    pat, f, gen_s, analyze_s = setup(args)
    M = args.systems
    streams = shard(rank, world, args.global_batch, args.scaling)
    B = len(streams)
    N, nnz_lower = pat.N, pat.K.nnz
    st = f.stats
    policy = policy_of(args)
    LOWER = nat.LAYOUT_SYMMETRIC_LOWER
    K, W = args.steps, args.warmup
    ks = [step_k(s, M) for s in range(K)]
    # warm-up walks the sequence backwards from its last (most refined) step, so the FGMRES
    # graphs and the straggler helpers' resume graphs are captured before the timed region
    wks = [M - 1 - (s % (M - 1)) for s in range(W)]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    host = {}
    for k in sorted(set(ks + wks)):
        items = gen_parallel(pat, [(k, q) for q in streams], min(threads, 16))
        host[k] = (np.stack([i[0] for i in items]), np.stack([i[1] for i in items]), items[0][2])
    gen_s += time.perf_counter() - t0
    t0 = time.perf_counter()
    dev = DeviceSystem(f, restart_m=10, device=local, batch=B)
    create_s = time.perf_counter() - t0
    stream = dev.stream
    with torch.cuda.stream(stream):
        dbat = {k: (torch.from_numpy(v).to(dev.device), torch.from_numpy(r).to(dev.device))
                for k, (v, r, _) in host.items()}
        dx = torch.empty((B, N), dtype=torch.float64, device=dev.device)
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev.device)
    stream.synchronize()
    handoff = not args.no_handoff

    def flush_l2():
        with torch.cuda.stream(stream):
            flush.fill_(1.0)

    def step_dev(k, pol):
        v, r = dbat[k]
        reps = dev.step(v, LOWER, r, dx, True, 10, 10, pol(host[k][2]), stats=True,
                        handoff=handoff)
        return reps if isinstance(reps, list) else [reps]

    def timed_steps(pol):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        out = []
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for s, k in enumerate(ks):
            flush_l2()
            ev[s][0].record(stream)
            reps = step_dev(k, pol)
            ev[s][1].record(stream)
            out.append([(r.iterations, r.converged, rr_of(r), r.handed_off, r.triggered)
                        for r in reps])
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ev], out

    for k in wks:
        step_dev(k, policy)
    launches0 = dev.launch_count()
    with Clocks(local) as clk:
        step_ms, recs = timed_steps(policy)
    launches = dev.launch_count() - launches0
    total_ms = reduce_max(float(np.sum(step_ms)), dist, dev.device)
    n_job = K * B * world
    value = total_ms / n_job

    def summarise(recs):
        its = np.array([[r[0] for r in step] for step in recs], dtype=float)
        conv = sum(r[1] for step in recs for r in step)
        rr = max(r[2] for step in recs for r in step)
        return {"mean_ir_iterations": float(its.mean()),
                "max_ir_iterations_per_step": [int(x) for x in its.max(axis=1)],
                "triggered": int(sum(r[4] for step in recs for r in step)),
                "handed_off": int(sum(r[3] for step in recs for r in step)),
                "converged": int(reduce_sum(conv, dist, dev.device)),
                "systems": n_job, "max_rr": float(reduce_max(rr, dist, dev.device))}

    check = summarise(recs)

    # ---- e2e through the public API from pinned host buffers (copies overlapped) ----
    hp = {k: (torch.from_numpy(v).pin_memory(), torch.from_numpy(r).pin_memory())
          for k, (v, r, _) in host.items()}
    hx = [torch.empty((B, N), dtype=torch.float64).pin_memory() for _ in range(2)]
    pipe = BatchPipeline(dev, LOWER)
    pipe.run([(hp[k][0], hp[k][1], hx[0], policy(host[k][2])) for k in wks])  # warm-up
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_reps = pipe.run([(hp[k][0], hp[k][1], hx[s % 2], policy(host[k][2]))
                         for s, k in enumerate(ks)])
    torch.cuda.synchronize()
    e2e_total = reduce_max((time.perf_counter() - t0) * 1e3, dist, dev.device)
    e2e_conv = sum(int(bool(q.converged)) for rp in e2e_reps for q in rp)
    e2e_value = e2e_total / n_job
    # the PCIe floor of the e2e leg: this box's pinned H2D bandwidth (one step's input size)
    h2d_bytes = 8 * B * (nnz_lower + N)
    hsrc = hp[ks[0]][0]
    with torch.cuda.stream(stream):
        ddst = torch.empty(hsrc.shape, dtype=torch.float64, device=dev.device)
    for _ in range(2):
        ddst.copy_(hsrc, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
        for _ in range(3):
            ddst.copy_(hsrc, non_blocking=True)
        b.record(stream)
    b.synchronize()
    h2d_gbs = 3 * hsrc.numel() * 8 / (a.elapsed_time(b) * 1e6)
    del ddst

    # ---- fixed delta = 1e-10 (the reference's RefinementConfig default order of magnitude) ----
    fixed = None
    if not args.no_fixed and args.tol == "barrier":
        fpol = policy_of(args, fixed=True)
        for k in wks:
            step_dev(k, fpol)
        fms, frecs = timed_steps(fpol)
        ftot = reduce_max(float(np.sum(fms)), dist, dev.device)
        fixed = {"delta": args.delta, "value": ftot / n_job, "unit": "ms/system",
                 "step_ms": [round(x, 3) for x in fms], **summarise(frecs)}

    # ---- per-kernel roofline on the batch (flushed L2) + the critical-path bound ----
    nL, nU = st["nnz_L"], st["nnz_U"]
    nnz_g = st["nnz_general"]
    pairs = st["update_pairs"]
    # algorithmic bytes: pattern/schedule once, values per system
    bytes_tri = (4 * (nL + nU) + 8 * (N + 1) * 2
                 + B * (8 * (nL + nU) + 8 * N + 12 * N + 16 * N + 12 * N))
    bytes_spmv = 4 * nnz_g + 8 * (N + 1) + B * (8 * nnz_g + 8 * N + 8 * N)
    bytes_ref = (4 * (nL + nU) + 4 * nU + 2 * pairs + 4 * pairs + 16 * nnz_g
                 + B * (8 * nnz_lower + 8 * nnz_g + 8 * (nL + nU + N) + 8 * (nL + nU)))

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

    with torch.cuda.stream(stream):  # internal-layout vectors: the kernels alone
        xb = torch.randn((N * dev.nbp(),), dtype=torch.float64, device=dev.device)
        yb = torch.empty_like(xb)
    t_tri = timed(lambda: dev.solve_native(xb, yb), args.kernel_reps)
    t_spmv = timed(lambda: dev.spmv_native(xb, yb), args.kernel_reps)
    t_ref = timed(lambda: dev.refactor_device(dbat[ks[-1]][0], LOWER), args.kernel_reps)
    peak, peak_kind = peaks()
    import ctypes
    hop_ns = ctypes.c_double()
    nat.check(nat.load().kkt_probe_hop_ns(local, 20000, ctypes.byref(hop_ns)), "kkt_probe_hop_ns")
    hop = float(hop_ns.value)
    lev_ref, lev_L, lev_U = st["refactor_levels"], st["L_levels"], st["U_levels"]
    cp = (lambda hops: hops * hop * 1e-6 if hop else None)
    kern = {
        "trisolve_pair": {"ms": t_tri, "bytes": bytes_tri, "GBs": bytes_tri / t_tri / 1e6,
                          "levels": lev_L + lev_U, "critical_path_ms": cp(lev_L + lev_U)},
        "spmv": {"ms": t_spmv, "bytes": bytes_spmv, "GBs": bytes_spmv / t_spmv / 1e6,
                 "hbm_floor_ms": bytes_spmv / peak / 1e6},
        "refactor": {"ms": t_ref, "bytes": bytes_ref, "GBs": bytes_ref / t_ref / 1e6,
                     "flops": st["refactor_flops"] * B,
                     "GFLOPs": st["refactor_flops"] * B / t_ref / 1e6,
                     "levels": lev_ref, "critical_path_ms": cp(lev_ref)},
    }
    for kd in kern.values():
        kd["hbm_floor_ms"] = kd["bytes"] / peak / 1e6
    its = np.array([[r[0] for r in step] for step in recs], dtype=float)
    max_iters = float(its.max(axis=1).mean()) if its.size else 0.0
    # time share per step: one solve per FGMRES iteration of the slowest system + the initial
    # solve; one refactorization; SpMV a few times per iteration
    share = {"trisolve_pair": t_tri * (1 + max_iters), "refactor": t_ref,
             "spmv": t_spmv * (max_iters + 3)}
    dom = max(share, key=share.get)
    kd = kern[dom]
    traffic = None  # the committed capture is of the default workload only
    same_workload = args.config == "activsg10k" and args.imbalance_frac == 1.0 and B == 64
    tp = os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")
    if not os.path.exists(tp):
        tp = os.path.join(ROOT, "profiles", "r1l_ncu_traffic.json")
    if same_workload and os.path.exists(tp):
        tk = json.load(open(tp))["kernels"]
        light = "k_b_refactor2" if "k_b_refactor2" in tk else "k_b_refactor"  # (two systems per lane)
        fam = {"refactor": [light, "k_b_refactor_tma<"], "spmv": ["k_b_spmv"],
               "trisolve_pair": ["k_b_trsv_grid<0,", "k_b_trsv_grid<1,", "k_trsv_blocked<0, 1,",
                                 "k_trsv_blocked<1, 1,"]}[dom]
        # a member ending in "<" or "," matches any instantiation of that template
        hit = [[k for k in tk if (k.startswith(f) if f.endswith(("<", ",")) else k == f)] for f in fam]
        if all(len(h) == 1 for h in hit):
            traffic = sum(tk[h[0]]["dram_read_bytes"] + tk[h[0]]["dram_write_bytes"] for h in hit)

    # ---- configs[2]: the single-system sequence latency (B = 1, barrier order) ----
    sequence = None
    if not args.no_single and rank == 0:
        from paper_2401_13926_b200.acopf import MU_STEP, system_rhs, system_values
        d1 = f.device(restart_m=10)
        sv = np.stack([system_values(pat, k, 0) for k in range(1, M)])
        sr = np.stack([system_rhs(pat, k, 0) for k in range(1, M)])
        sd = [policy(10.0 ** (-MU_STEP * k)) for k in range(1, M)]
        with torch.cuda.stream(d1.stream):
            sv_t = torch.from_numpy(sv).to(d1.device)
            sr_t = torch.from_numpy(sr).to(d1.device)
            sx_t = torch.empty(N, dtype=torch.float64, device=d1.device)
        # warm-up with the timed call's arguments: the last (IR-triggering) systems first, so
        # every FGMRES graph variant the timed loop uses is captured before it
        for k in (M - 2, M - 3, 0, 1, 2):
            d1.step(sv_t[k], LOWER, sr_t[k], sx_t, True, 10, 10, sd[k], stats=True)
        lat, its1, rr1 = [], [], []
        for k in range(M - 1):
            with torch.cuda.stream(d1.stream):
                flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(d1.stream)
            rep = d1.step(sv_t[k], LOWER, sr_t[k], sx_t, True, 10, 10, sd[k], stats=True)
            b.record(d1.stream)
            b.synchronize()
            lat.append(a.elapsed_time(b))
            its1.append(rep.iterations)
            rr1.append(rr_of(rep))
        # e2e: host (pinned) values and rhs in, x out through kkt_dev_step
        pv = torch.from_numpy(sv).pin_memory().numpy()
        pr = torch.from_numpy(sr).pin_memory().numpy()
        px = torch.empty((M - 1, N), dtype=torch.float64).pin_memory().numpy()
        e2e1 = []
        for k in (M - 2, 0):  # warm the host-buffer path too (its first call sets up staging)
            d1.step(pv[k], LOWER, pr[k], px[k], False, 10, 10, sd[k])
        for k in range(M - 1):
            with torch.cuda.stream(d1.stream):
                flush.fill_(1.0)
            d1.stream.synchronize()
            t0 = time.perf_counter()
            d1.step(pv[k], LOWER, pr[k], px[k], False, 10, 10, sd[k])
            e2e1.append((time.perf_counter() - t0) * 1e3)
        cpu1 = None
        if not args.no_cpu_baseline:
            items = [(sv[k], sr[k], 10.0 ** (-MU_STEP * (k + 1))) for k in range(M - 1)]
            _, _, per = cpu_port_run(f, pat.K, items, policy, 1)
            cpu1 = float(np.mean(per) * 1e3)
        mean1, e2e_mean1 = float(np.mean(lat)), float(np.mean(e2e1))
        sequence = {
            "workload": f"{args.config} sequence (configs[2] shape at activsg10k): systems 1.."
                        f"{M - 1} of value stream 0 in barrier order on a single-system handle "
                        "(refactor + lu_solve + refine_fgmres each)",
            "ms_per_system_mean": mean1, "ms_median": float(np.median(lat)),
            "e2e_ms_per_system_mean": e2e_mean1,
            "ms_per_system": [round(x, 3) for x in lat],
            "e2e_ms_per_system": [round(x, 3) for x in e2e1],
            "ir_iterations": its1, "max_rr": float(max(rr1)),
            "cpu_single_thread_ms_mean": cpu1,
            "speedup_vs_cpu_1t": (cpu1 / mean1) if cpu1 else None,
            "speedup_e2e_vs_cpu_1t": (cpu1 / e2e_mean1) if cpu1 else None,
            "schedule": d1.info()}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        qs = streams[:8]
        items = [(k, q) for q in qs for k in ks]
        systems = gen_parallel(pat, items, min(threads, 16))
        wall, n_sys, per = cpu_port_run(f, pat.K, systems, policy, 1, budget_s=args.cpu_seconds,
                                        round_len=len(ks))
        cpu = {"value": float(np.mean(per) * 1e3), "unit": "ms/system", "cores": 1, "kind": "port",
               "sample": f"{n_sys} of the timed systems (value streams {qs[0]}.. x barrier steps "
                         f"{ks[0]}..{max(ks)}, whole rounds of the {len(ks)} steps), "
                         f"refactorize+lu_solve+refine_fgmres, single thread, "
                         f"oracle/kkt_oracle.c, {wall:.1f}s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "ms/system", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": False, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": workload_desc(args, world),
                "barrier_steps": ks, "global_batch": args.global_batch,
                "systems_per_gpu": B, "value_streams_rank0": [streams[0], streams[-1]],
                "N": N, "nnz_lower": nnz_lower, "nnz_general": nnz_g,
                "nnz_L": nL, "nnz_U": nU, "refactor_flops_per_system": st["refactor_flops"],
                "levels_refactor_L_U": [lev_ref, lev_L, lev_U],
                "offdiag_pivots": st["offdiag_pivots"], "imbalance_frac": args.imbalance_frac,
                "update_pairs_per_system": st["update_pairs"],
                "tolerance": ("delta(mu)=clamp(1e-2*mu,1e-10,1e-8) per system"
                              if args.tol == "barrier" else f"{args.delta}"),
                "straggler_handoff": handoff,
                "l2": "flushed between steps (256 MiB write, excluded from timing); inputs "
                      "of a step (490 MB at 64 systems) exceed L2",
                "e2e_note": "pinned host inputs H2D + x D2H per step, overlapped with "
                            "neighbouring steps (pipeline.BatchPipeline)",
                "analyze_s": analyze_s, "device_create_s": create_s, "generate_s": gen_s,
                "parallelism": f"{world} GPU(s), one process each, independent shards "
                               "(no data-path collective)",
                "step_ms": [round(x, 3) for x in step_ms],
                "schedule": dev.info(),
            },
            "check": check,
            "e2e": {"value": e2e_value, "unit": "ms/system",
                    "h2d_bytes_per_step": h2d_bytes,
                    "d2h_bytes_per_step": 8 * B * N,
                    "h2d_gbs_measured": h2d_gbs,
                    "pcie_floor_ms_per_system": h2d_bytes / (h2d_gbs * 1e6) / B,
                    "converged_rank0": e2e_conv, "systems_rank0": B * len(ks)},
            "sequence": sequence,
            "fixed_delta": fixed,
            "roofline": {"kernel": dom, "bound": "hbm", "achieved": kd["GBs"], "peak": peak,
                         "unit": "GB/s", "frac": kd["GBs"] / peak, "traffic": traffic,
                         "algorithmic_bytes": kd["bytes"], "peak_kind": peak_kind,
                         "critical_path": {"levels": kd.get("levels"), "hop_ns": hop,
                                           "bound_ms": kd.get("critical_path_ms"),
                                           "measured_ms": kd["ms"],
                                           "hbm_floor_ms": kd["hbm_floor_ms"]},
                         "note": "refactor/trisolve are DAG chains: the critical-path bound "
                                 "(levels x measured inter-SM hop) and the HBM floor are both "
                                 "stated; the batch amortises the chain (DESIGN.md §5)"},
            "kernels": kern,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
        if check["converged"] != check["systems"] or (fixed and fixed["converged"] != fixed["systems"]):
            print("bench: a timed system did not converge", file=sys.stderr)
            raise SystemExit(1)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
