"""Multi-GPU host logic of bench.py: one process per GPU, every rank
factors its own independent instance of the workload (weak scaling over independent problems,
no data-path collective); the step time is the maximum over ranks of device-event times."""
from __future__ import annotations

import dataclasses


def instance_config(cfg, rank: int):
    """Rank r > 0 draws its own instance: same distribution, kernel, leaf, tol and nrhs, seed
    offset by 1000 r (rank 0 keeps the BASELINE seed)."""
    return cfg if rank == 0 else dataclasses.replace(cfg, seed=cfg.seed + 1000 * rank)


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


def aggregate_throughput(n_per_rank, world: int, seconds_max: float):
    """Whole-job unknowns/s: all ranks' unknowns over the slowest rank's time."""
    return world * n_per_rank / seconds_max
