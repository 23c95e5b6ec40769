"""Multi-process host logic of the sharded path (world size 2, gloo, CPU)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_03067_b200.dist import gather_compression, gather_tables, shard_units


@pytest.mark.parametrize("n,world", [(32, 1), (32, 2), (32, 8), (80, 3), (5, 8), (640, 8)])
def test_shard_units_partition(n, world):
    seen = []
    sizes = []
    for r in range(world):
        rg = shard_units(n, world, r)
        seen.extend(rg)
        sizes.append(len(rg))
    assert seen == list(range(n))
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        units = shard_units(5, world, rank)
        nb = 16
        before = torch.full((len(units),), nb, dtype=torch.int64)
        after = torch.tensor([nb - 1 - u for u in units], dtype=torch.int64)
        stats = gather_compression(before, after)
        table = torch.stack([torch.arange(nb, dtype=torch.int32) * (u + 1) for u in units])
        tables = gather_tables(table, dst=0)
        if rank == 0:
            q.put((stats.blocks_before, stats.blocks_after, stats.per_rank_after,
                   [t.tolist() for t in tables]))
    finally:
        dist.destroy_process_group()


def test_gather_stats_and_tables_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    before, after, per_rank, tables = q.get(timeout=10)
    assert before == 5 * 16
    assert after == sum(16 - 1 - u for u in range(5))
    assert per_rank == [sum(15 - u for u in shard_units(5, 2, r)) for r in range(2)]
    flat = [row for t in tables for row in t]
    assert flat == [[j * (u + 1) for j in range(16)] for u in range(5)]
