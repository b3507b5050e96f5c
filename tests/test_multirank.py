"""The N > 1 path of bench.py on CPU (gloo, world_size 2): ranks shard independent systems
(distinct value streams, no data-path collective), each rank's systems go through the same
per-system pipeline (here the CPU oracle restatement, the GPU's checker), and the job time is
the max over ranks.  Mirrors what `torchrun --nproc-per-node N bench.py` does on GPUs."""

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


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import oracle
        from paper_2401_13926_b200 import factorize, to_general
        from paper_2401_13926_b200.acopf import build_pattern, system_rhs, system_values
        from paper_2401_13926_b200.sparse import expand_pattern
        ks = [bench.step_k(s, 20) for s in range(3)]
        mine = bench.rank_systems(rank, 2, ks)
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        pat = build_pattern(40, 0)
        K0 = pat.K.with_values(system_values(pat, 0, 0))
        f, _ = factorize(to_general(K0))
        ex = expand_pattern(K0)
        arrays = dict(row_perm=f.row_perm.perm, col_perm=f.col_perm.perm, Lp=f._Lp, Li=f._Li,
                      Lx=f._Lx, Up=f._Up, Ui=f._Ui, Ux=f._Ux, Udiag=f._Udiag,
                      so_ptr=f._so_ptr, so_data=f._so_data, ap_ptr=f._ap_ptr,
                      a_src=f._a_src, a_tgt=f._a_tgt)
        of = oracle.OracleFactors(arrays, ex.general.row_ptr)
        sols = []
        for k, seed in mine:
            of.refactorize(system_values(pat, k, seed)[ex.src])
            sols.append(of.lu_solve(system_rhs(pat, k, seed)))
        t_mine = 1.0 + rank  # stand-in per-rank time
        t_job = bench.reduce_max(t_mine, dist, "cpu")
        out.put((rank, allv, t_job, [float(np.linalg.norm(x)) for x in sols]))
    finally:
        dist.destroy_process_group()


def test_two_ranks_shard_disjoint_systems_and_take_max_time():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    allv = res[0][1]
    assert res[1][1] == allv                                  # same view on both ranks
    assert not set(allv[0]) & set(allv[1])                    # disjoint shards
    assert len(allv[0]) == len(allv[1]) == 6
    assert res[0][2] == res[1][2] == 2.0                      # max over ranks
    assert all(np.isfinite(v) and v > 0 for r in res for v in r[3])
