"""world_size-2 gloo run of the scan-sharding logic used by bench.py (CPU)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_10319_b200.sharding import max_over_ranks, shard_seeds
    seeds = shard_seeds(rank, world, 8)
    gathered = [None] * world
    dist.all_gather_object(gathered, seeds)
    t = max_over_ranks(1.5 + rank)
    if rank == 0:
        q.put((gathered, t))
    dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, t = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert gathered == [list(range(0, 8)), list(range(8, 16))]
    assert t == 2.5  # max over ranks


def _orchestrate(rank, world, port, q):
    """The bench's multi-GPU data path on CPU: a fixed batch of scans (strong
    scaling, config 5) assigned by LPT on voxel count, each rank runs its
    scans through a forward stub, and the per-scan outputs are gathered to
    rank 0 -- the path's only data collective."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_10319_b200.sharding import gather_outputs, lpt_assign
    sizes = [50 + 13 * ((7 * i) % 11) for i in range(12)]          # voxels per scan
    mine = lpt_assign(sizes, world)[rank]

    def forward_stub(scan):                                       # (rows, 3) logits
        g = torch.Generator().manual_seed(scan)
        return torch.randn((sizes[scan], 3), generator=g, dtype=torch.float16)

    got = gather_outputs({s: forward_stub(s) for s in mine})
    if rank == 0:
        # numpy arrays travel by value (torch tensors would be shared through
        # a file-descriptor socket that can vanish once this process exits)
        q.put({k: v.numpy().copy() for k, v in got.items()})
    else:
        assert got is None
    dist.destroy_process_group()


def test_two_rank_shard_forward_gather_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_orchestrate, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    sizes = [50 + 13 * ((7 * i) % 11) for i in range(12)]
    assert sorted(got) == list(range(12))
    for s in range(12):
        g = torch.Generator().manual_seed(s)
        assert torch.equal(torch.from_numpy(got[s]),
                           torch.randn((sizes[s], 3), generator=g, dtype=torch.float16))


def test_gather_outputs_single_process_is_identity():
    from paper_2204_10319_b200.sharding import gather_outputs
    x = {3: torch.ones(2, 2)}
    assert gather_outputs(x) == x


def test_lpt_balances():
    from paper_2204_10319_b200.sharding import lpt_assign, shard_seeds
    a = lpt_assign([120, 130, 90, 125, 100, 110, 95, 127], 4)
    assert sorted(i for r in a for i in r) == list(range(8))
    loads = [sum([120, 130, 90, 125, 100, 110, 95, 127][i] for i in r) for r in a]
    assert max(loads) - min(loads) <= 40
    with pytest.raises(ValueError):
        shard_seeds(2, 2, 8)
