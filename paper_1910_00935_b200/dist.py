"""Episode sharding and the one collective of the path.

The differentiable MLS-MPM step shards only across independent episodes: each rank
(one process per GPU) simulates its own episodes, and the only exchange is an
all-reduce(SUM) of the gradient of the parameters the episodes share (the controller
weights theta, or a shared uniform initial velocity) once per optimisation iteration.
Timing is the max over ranks.  These helpers are backend-agnostic (NCCL on GPUs, gloo
in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def episode_shard(total: int, rank: int, world: int) -> range:
    """Contiguous block of episode indices of `rank` (sizes differ by at most one)."""
    if total < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard request")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def allreduce_shared_grad(grad: torch.Tensor) -> torch.Tensor:
    """Sum the shared-parameter gradient over ranks, in place (no-op without a group)."""
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(grad, op=dist.ReduceOp.SUM)
    return grad


def max_over_ranks(value: float, device: torch.device | str = "cpu") -> float:
    """Max of a per-rank scalar (e.g. elapsed device ms) over all ranks."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_scaling_value(units_per_rank: float, world: int, ms_max: float) -> float:
    """Whole-job throughput: units processed by all ranks / max-over-ranks time."""
    return units_per_rank * world / (ms_max / 1e3)
