"""Multi-GPU plumbing for the speculation path: one process per GPU.

Requests are independent units, so the path shards by request
with no data-path collective: rank r serves its own slice of the request list
on its own GPU with its own model replicas ("replicas only" for the cfg2
workload, weak scaling).  The only collectives are control-plane: a barrier
around timed regions and max/sum reductions of the per-rank timings and token
counts (device-agnostic: NCCL on GPU ranks, gloo in the CPU tests).
"""
from __future__ import annotations

import os
from typing import Sequence

import torch


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_requests(requests: Sequence, rank: int, world_size: int) -> list:
    """Contiguous, balanced slice of the request list for `rank` (every request
    lands on exactly one rank; slice sizes differ by at most one)."""
    n = len(requests)
    lo = rank * n // world_size
    hi = (rank + 1) * n // world_size
    return list(requests[lo:hi])


def _reduce(x: float, op, device) -> float:
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x: float, device="cpu") -> float:
    import torch.distributed as dist
    return _reduce(x, dist.ReduceOp.MAX if dist.is_available() else None, device)


def sum_over_ranks(x: float, device="cpu") -> float:
    import torch.distributed as dist
    return _reduce(x, dist.ReduceOp.SUM if dist.is_available() else None, device)


def sync_time_fn(device="cpu"):
    """The tensor-parallel engine's `sync_time`: a rank's selector time ->
    the max over ranks (fp64 all-reduce), so every rank feeds its selector
    the same MonitorSample.t_llm and takes the same decisions (rounds.py)."""
    import torch.distributed as dist

    def sync(ms: float) -> float:
        t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return sync


def barrier() -> None:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
