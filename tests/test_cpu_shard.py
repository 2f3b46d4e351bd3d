"""CPU tests of the element-sharding host logic (shard.py): balanced contiguous
slices, and the output gather / all-gather over torch.distributed with gloo at
world_size 2 and 3 (uneven slices, several dtypes and row shapes) -- the same
code that moves the evaluated shares over NCCL on a multi-GPU box."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2006_04593_b200 import shard


@pytest.mark.parametrize("total", [0, 1, 5, 7, 64, 1001])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_bounds_partition(total, world):
    spans = [shard.shard_bounds(total, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (lo, hi), (lo2, _) in zip(spans, spans[1:]):
        assert hi == lo2
    sizes = [hi - lo for lo, hi in spans]
    assert max(sizes) - min(sizes) <= 1


def test_shard_bounds_errors():
    with pytest.raises(ValueError):
        shard.shard_bounds(10, 2, 2)
    with pytest.raises(ValueError):
        shard.shard_bounds(10, 0, 0)
    with pytest.raises(ValueError):
        shard.shard_bounds(-1, 0, 1)


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _global(total):
    g = torch.Generator().manual_seed(1234)
    u64 = torch.randint(0, 1 << 62, (total,), generator=g, dtype=torch.int64).view(torch.uint64)
    u8 = torch.randint(0, 256, (total, 16), generator=g, dtype=torch.int64).to(torch.uint8)
    flags = torch.randint(0, 2, (total,), generator=g).bool()
    return u64, u8, flags


def _worker(rank, world, port, total, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard.shard_bounds(total, rank, world)
        u64, u8, flags = _global(total)
        got = shard.gather_shards(u64[lo:hi], total, dst=world - 1)
        got8 = shard.all_gather_shards(u8[lo:hi], total)
        gotb = shard.gather_shards(flags[lo:hi], total, dst=0)
        ring = shard.gather_ring(u64[lo:hi], 64, total, dst=None)
        ok = torch.equal(got8, u8) and torch.equal(ring.view(torch.int64), u64.view(torch.int64))
        if rank == world - 1:
            ok = ok and torch.equal(got.view(torch.int64), u64.view(torch.int64))
        else:
            ok = ok and got is None
        if rank == 0:
            ok = ok and torch.equal(gotb, flags)
        with pytest.raises(ValueError):   # wrong slice length
            shard.gather_shards(torch.zeros(hi - lo + 1, dtype=torch.uint64), total)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 1), (3, 1000)])
def test_gather_shards_gloo(world, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
    assert all(p.exitcode == 0 for p in procs)
