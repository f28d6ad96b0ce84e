"""world_size-2 gloo test of the multi-GPU host logic (paper_2301_12704_b200/dist.py) used by
bench.py under torchrun: independent per-rank instances, max-over-ranks timing, whole-job
throughput.  Each rank also solves its own small instance with the oracle and the ranks agree
on the worst residual through the same all-reduce (CPU only)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2301_12704_b200 import dist as D, workloads as W
    from oracle import dense
    from oracle.factor import AIFMM
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = W.CONFIGS[1]
    ci = D.instance_config(cfg, rank)
    pts, b = W.make(ci, n=600, nrhs=1)
    o = AIFMM(pts, ci.kernel_id, ci.kparams, 32, 1e-8).factor()
    x = o.solve(b)
    res = dense.residual(pts, ci.kernel_id, ci.kparams, x, b)
    mx = D.max_over_ranks([1.0 + rank, 10.0 - rank, res])
    q.put((rank, ci.seed, float(pts[0, 0]), mx, D.aggregate_throughput(600, world, mx[0])))
    dist.destroy_process_group()


def test_two_rank_gloo_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, s0, p0, m0, v0), (r1, s1, p1, m1, v1) = out
    assert s0 == 1 and s1 == 1001 and p0 != p1          # independent instances
    assert m0 == m1 and m0[0] == 2.0 and m0[1] == 10.0   # max over ranks, identical on both
    assert m0[2] <= 1e-6                                  # both instances solved
    assert v0 == v1 == 2 * 600 / 2.0
