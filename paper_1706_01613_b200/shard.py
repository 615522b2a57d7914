"""Sharding of the hexahedra across ranks (one process per GPU).

The hexes are independent (the check takes one element's
8 nodes and returns its validity), so the path partitions with no data-path
exchange.  Two modes:

* weak scaling (``bench.py``): every rank checks its own ``n`` hexes, rank r
  the synthetic hexes ``r*n .. r*n+n-1`` of the configuration's stream;
* strong scaling: ``n_total`` hexes split into contiguous, balanced ranges.

The only collectives are host-side bookkeeping: the barrier around the timed
region, the max over ranks of the device time, and the sum of the verdict
counters.  They run on whatever backend ``torch.distributed`` was initialised
with (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

__all__ = ["weak_shard", "strong_shard", "max_over_ranks", "sum_over_ranks", "barrier"]


def weak_shard(n_per_rank: int, rank: int) -> tuple[int, int]:
    """(start, count) of rank ``rank`` when every rank processes ``n_per_rank`` hexes."""
    if n_per_rank < 0 or rank < 0:
        raise ValueError("n_per_rank and rank must be >= 0")
    return rank * n_per_rank, n_per_rank


def strong_shard(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count): contiguous ranges whose sizes differ by at most one hex."""
    if world <= 0 or not 0 <= rank < world or n_total < 0:
        raise ValueError("need world > 0, 0 <= rank < world, n_total >= 0")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _device():
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(x: float) -> float:
    """Max of a host float over all ranks (identity without a process group)."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values: list[int]) -> list[int]:
    """Element-wise sum of integer counters over all ranks."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return [int(v) for v in values]
    import torch
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(v) for v in t.tolist()]


def barrier() -> None:
    dist = _dist()
    if dist is not None and dist.get_world_size() > 1:
        dist.barrier()
