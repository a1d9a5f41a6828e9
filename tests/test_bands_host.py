"""CPU tests of the multi-GPU host logic: band geometry, batch sharding, and the band exchange over a
world_size-2 gloo process group (the same code path NCCL drives between B200s)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1609_05722_b200 import bands


def test_tile_grid_and_partition():
    tx, ty = bands.tile_grid(5, 8192, 8192)
    assert (tx, ty) == (-(-8192 // 60), -(-8192 // 32))
    for n in (1, 2, 3, 4, 8):
        parts = bands.partition_tile_rows(ty, n)
        assert parts[0][0] == 0 and parts[-1][1] == ty
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        bands.partition_tile_rows(3, 4)


@pytest.mark.parametrize("m", [3, 5, 7])
def test_band_geometry_covers_image(m):
    H, W = 1000, 300
    _, ty = bands.tile_grid(m, H, W)
    r = m // 2
    parts = bands.partition_tile_rows(ty, 4)
    prev_end = 0
    for k, (t0, t1) in enumerate(parts):
        d = bands.band_geometry(m, 2, H, W, t0, t1)
        assert d.row0 == prev_end and d.row1 > d.row0 and d.halo == 2 * r
        assert d.lrow0 == max(0, d.row0 - 2 * r)
        assert d.lrow0 + d.Hl == min(H, d.row1 + 2 * r)
        prev_end = d.row1
    assert prev_end == H
    # the last tile row is pulled up to own >= r rows (symmetric fold stays in one tile)
    last = bands.band_geometry(m, 1, H, W, ty - 1, ty)
    assert last.row1 - last.row0 >= r


def test_shard_batch_partitions():
    for n, world in ((256, 8), (10, 3), (5, 5)):
        got = []
        for r in range(world):
            s = bands.shard_batch(n, r, world)
            got.extend(range(n)[s])
        assert got == list(range(n))


def _exchange_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = bands.DistExchange()
        # per-rank partial chunks of different lengths inside one global array
        chunks = [(0, 5), (5, 3)]
        off, cnt = chunks[rank]
        partials = torch.full((8,), -1.0, dtype=torch.float64)
        partials[off:off + cnt] = torch.arange(off, off + cnt, dtype=torch.float64) * 10
        send = torch.stack([torch.full((6,), 100.0 * rank + 1), torch.full((6,), 100.0 * rank + 2)])
        recv = torch.zeros(2, 6)
        ex.exchange_arrays(partials, slice(off, off + cnt), chunks, send, recv)
        q.put((rank, partials.tolist(), recv.tolist()))
    finally:
        dist.destroy_process_group()


def test_dist_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 2000
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (a, b)) for r, a, b in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = [float(10 * i) for i in range(8)]
    assert res[0][0] == full and res[1][0] == full
    # rank 0 (top band): dir 1 receives rank 1's dir 0 (its first owned rows); dir 0 untouched
    assert res[0][1][1] == [101.0] * 6 and res[0][1][0] == [0.0] * 6
    # rank 1 (bottom band): dir 0 receives rank 0's dir 1 (its last owned rows)
    assert res[1][1][0] == [2.0] * 6 and res[1][1][1] == [0.0] * 6
