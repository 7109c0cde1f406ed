"""Multi-GPU plumbing for batched throughput: independent
encrypted requests are partitioned across ranks with no collective on the
data path; the only collectives are a barrier and the max-over-ranks of the
device-timed elapsed seconds. Backend-agnostic (nccl on GPUs, gloo in tests).
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(total: int, world_size: int, rank: int) -> range:
    """Contiguous, disjoint image range of `rank` (weak scaling uses
    total = world_size * per_rank)."""
    if not 0 <= rank < world_size:
        raise ValueError("rank out of range")
    lo = total * rank // world_size
    hi = total * (rank + 1) // world_size
    return range(lo, hi)


def barrier(world_size: int) -> None:
    if world_size > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(value: float, world_size: int, device: str = "cuda") -> float:
    if world_size == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, world_size: int, device: str = "cuda") -> float:
    if world_size == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
