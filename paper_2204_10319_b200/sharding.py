"""Scan-level sharding across ranks: scans are independent,
so each rank owns a disjoint, contiguous block of scan seeds and there is no
collective in the data path.  The only cross-rank operation is the timing
reduction (max over ranks)."""

from __future__ import annotations


def shard_seeds(rank: int, world: int, per_rank: int, first: int = 0) -> list[int]:
    """Seeds of the scans rank `rank` processes (weak scaling: `per_rank` each)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    start = first + rank * per_rank
    return list(range(start, start + per_rank))


def lpt_assign(sizes, world: int) -> list[list[int]]:
    """Longest-processing-time assignment of scans (by voxel count) to ranks,
    for strong-scaling runs over a fixed scan set."""
    loads = [0] * world
    out = [[] for _ in range(world)]
    for i in sorted(range(len(sizes)), key=lambda i: -sizes[i]):
        r = min(range(world), key=lambda r: loads[r])
        out[r].append(i)
        loads[r] += sizes[i]
    return out


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank time (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
