"""The N > 1 path of bench.py on CPU (gloo, world_size 2 and 4).

configs[4] — one global batch of 64 independent systems per step, split 64/G per GPU:
* `bench.shard` partitions the global batch into disjoint, equal, contiguous shards whose
  union is the whole job for G = 1, 2, 4, 8 (strong scaling), and gives every rank its own 64
  distinct value streams under --scaling weak;
* on real ranks (gloo here, NCCL on GPUs) every rank takes its shard, its systems go through
  the per-system pipeline (here the CPU oracle restatement, the GPU's checker) with NO data-path
  collective, and the job's time is the max over ranks (bench.reduce_max) while convergence
  counts add up (bench.reduce_sum).
"""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_strong_shards_partition_the_global_batch(world):
    import bench
    shards = [bench.shard(r, world, 64, "strong") for r in range(world)]
    assert all(len(s) == 64 // world for s in shards)
    flat = [q for s in shards for q in s]
    assert sorted(flat) == list(range(64)) == bench.job_streams(world, 64, "strong")
    assert all(s == list(range(s[0], s[0] + len(s))) for s in shards)  # contiguous


def test_weak_shards_are_distinct():
    import bench
    shards = [set(bench.shard(r, 4, 64, "weak")) for r in range(4)]
    assert all(len(s) == 64 for s in shards)
    assert len(set.union(*shards)) == 256


def test_uneven_split_is_rejected():
    import bench
    with pytest.raises(SystemExit):
        bench.shard(0, 3, 64, "strong")


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2401_13926_b200 import factorize, to_general
        from paper_2401_13926_b200.acopf import build_pattern, system_values
        streams = bench.shard(rank, world, 8, "strong")
        allv = [None] * world
        dist.all_gather_object(allv, streams)
        pat = build_pattern(40, 0)
        K0 = pat.K.with_values(system_values(pat, 0, 0))
        f, _ = factorize(to_general(K0))
        ks = [bench.step_k(s, 20) for s in range(3)]
        systems = [bench.make_batch(pat, streams, k) for k in ks]
        items = [(v[i], r[i], mu) for v, r, mu in systems for i in range(len(streams))]
        wall, done, per = bench.cpu_port_run(f, pat.K, items, bench.policy_of(bench.parse([])), 1)
        t_job = bench.reduce_max(1.0 + rank, dist, "cpu")
        n_job = bench.reduce_sum(done, dist, "cpu")
        out.put((rank, allv, t_job, n_job, done))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_process_their_shard_and_take_max_time(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    allv = res[0][1]
    assert all(r[1] == allv for r in res)                       # same view on every rank
    assert sorted(q for s in allv for q in s) == list(range(8))  # the 8-system job, split 8/G
    assert all(r[2] == float(world) for r in res)               # max over ranks
    assert all(r[3] == 3 * 8 for r in res)                      # every system of 3 steps, once
    assert all(r[4] == 3 * 8 // world for r in res)
