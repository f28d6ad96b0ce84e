"""world_size-2 gloo test of the multi-GPU host logic bench.py runs under torchrun
(paper_2301_12704_b200/dist.py): rank 0's NCCL unique id reaches every rank unchanged,
device times are maxed over ranks identically everywhere, and the strong-scaling throughput is
the whole problem over the slowest rank.  The data path itself (ownership split, exchanges) is
covered on the GPU by tests/test_gpu_dist.py with in-process ranks."""
import os
import socket

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
    from paper_2301_12704_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = D.share_unique_id(bytes(range(128)) if rank == 0 else None)
    mx = D.max_over_ranks([1.0 + rank, 10.0 - rank])
    q.put((rank, uid, mx, D.strong_throughput(1 << 20, mx[0])))
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
    (r0, u0, m0, v0), (r1, u1, m1, v1) = out
    assert u0 == u1 == bytes(range(128))                 # the library's NCCL id reached rank 1
    assert m0 == m1 == [2.0, 10.0]                        # max over ranks, identical on both
    assert v0 == v1 == (1 << 20) / 2.0                    # one problem, slowest rank's time


def test_single_process_identity():
    from paper_2301_12704_b200 import dist as D
    assert D.share_unique_id(b"x" * 128) == b"x" * 128
    assert D.max_over_ranks([3.0]) == [3.0]
    with pytest.raises(AssertionError):
        D.share_unique_id(None)
