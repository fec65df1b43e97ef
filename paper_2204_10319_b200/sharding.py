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


def gather_rows(local, rows_per_rank: list, dst: int = 0):
    """Gather each rank's (rows, C) result to ``dst`` when every rank's row
    count is already known (the bench: the same scans every step): one
    ``torch.distributed.gather`` of a buffer padded to the largest count, no
    host round trip.  Returns the per-rank row blocks on ``dst``, None
    elsewhere."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    cap = max(max(rows_per_rank), 1)
    if local.shape[0] == cap:
        flat = local.contiguous()
    else:
        flat = torch.zeros((cap, local.shape[1]), dtype=local.dtype, device=local.device)
        flat[: local.shape[0]] = local
    bufs = [torch.empty_like(flat) for _ in range(world)] if rank == dst else None
    dist.gather(flat, bufs, dst=dst)
    if rank != dst:
        return None
    return [b[:n] for b, n in zip(bufs, rows_per_rank)]


def gather_outputs(outputs: dict, dst: int = 0) -> dict | None:
    """The path's one data collective (BASELINE north_star: "no collective
    beyond the final output gather"): every rank's per-scan results
    ``{scan_id: (rows, C) tensor}`` are gathered to rank ``dst``, which gets
    ``{scan_id: tensor}`` for the whole batch (None on the other ranks).

    One flat buffer per rank (its scans concatenated, padded to the largest
    rank's row count) through ``torch.distributed.gather`` — NCCL over
    NVLink for CUDA tensors, gloo for host tensors — plus a gather of the
    (scan_id, rows) index.  Identity when not distributed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(outputs)
    rank, world = dist.get_rank(), dist.get_world_size()
    ids = sorted(outputs)
    index = [(i, int(outputs[i].shape[0])) for i in ids]
    ref = next(iter(outputs.values())) if outputs else None
    meta = [None] * world
    dist.all_gather_object(meta, (index, None if ref is None else (ref.shape[1], str(ref.dtype))))
    cols_dtype = next((m[1] for m in meta if m[1] is not None), None)
    if cols_dtype is None:
        return {} if rank == dst else None
    cols = cols_dtype[0]
    dtype = getattr(torch, cols_dtype[1].replace("torch.", ""))
    device = ref.device if ref is not None else (
        torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl"
        else torch.device("cpu"))
    rows = [sum(n for _, n in m[0]) for m in meta]
    local = torch.cat([outputs[i] for i in ids]) if ids else \
        torch.zeros((0, cols), dtype=dtype, device=device)
    bufs = gather_rows(local, rows, dst)
    if rank != dst:
        return None
    out = {}
    for r, (index_r, _) in enumerate(meta):
        o = 0
        for i, n in index_r:
            out[i] = bufs[r][o:o + n]
            o += n
    return out
