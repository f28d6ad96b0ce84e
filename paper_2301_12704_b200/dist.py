"""Multi-GPU host logic of bench.py: one process per GPU, all ranks factor the
same workload together through the library's subtree split (include/aifmm.h aifmm_dist_init;
the data path's collectives are NCCL calls inside libaifmm.so).  Here: handing the library's
NCCL unique id from rank 0 to the others, max-over-ranks device times, and the strong-scaling
throughput."""
from __future__ import annotations


def share_unique_id(uid: bytes | None) -> bytes:
    """Rank 0 passes its id (128 bytes), the others None; every rank returns rank 0's id
    (torch.distributed.broadcast_object_list over the default group; identity without one)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        assert uid is not None
        return uid
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    assert isinstance(obj[0], (bytes, bytearray)) and len(obj[0]) == 128, "bad NCCL unique id"
    return bytes(obj[0])


def max_over_ranks(values, device=None):
    """Element-wise maximum of a list of floats over all ranks (identity without a process
    group).  Uses the default group's backend (nccl on the GPU box, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def strong_throughput(n_total, seconds_max: float):
    """Whole-job unknowns/s of one problem of n_total unknowns solved by all ranks together:
    n_total over the slowest rank's time."""
    return n_total / seconds_max
