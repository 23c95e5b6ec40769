"""Layer-sharded fusion across ranks: two processes share
cuda:0 over gloo (this sandbox has one GPU per call; the NCCL path is the same code
with CUDA tensors), each fuses its dist.shard_units layers, all-gathers the block
counts and gathers the remapped tables to rank 0. The result must equal a single
run over all layers: same tables, refcount-derived CR, per-rank counts."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


SHAPE = dict(L=5, B=8, p=32, t=16, h=2, d=128)


def _cache(host: bool):
    from paper_2601_03067_b200.workload import synthetic_kv

    d = SHAPE
    Kt, Vt = synthetic_kv(d["L"], d["B"], d["p"], d["t"], d["h"], d["d"], dtype=torch.bfloat16, seed=41)
    dims = K.CacheDims(**d)
    if host:
        return K.PagedKvCache(dims, Kt.cpu().pin_memory(), Vt.cpu().pin_memory(), defer_upload=True)
    return K.PagedKvCache(dims, Kt, Vt)


def _worker(rank, world, port, host, head_mode, q):
    import torch.distributed as dist

    from paper_2601_03067_b200.dist import fuse_batch_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = fuse_batch_sharded(_cache(host), K.FusionConfig(threshold=0.8, head_mode=head_mode))
        layers = [o.report.layer for o in res.outcomes]
        if rank == 0:
            q.put((list(res.layers), layers, res.stats.blocks_before, res.stats.blocks_after,
                   res.stats.per_rank_after, [t.tolist() for t in res.tables]))
        else:
            q.put((list(res.layers), layers, None, None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("host,head_mode", [(False, "folded"), (True, "folded"), (False, "per_head")])
def test_sharded_equals_single_run(host, head_mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, host, head_mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda x: x[0][0])
    full = K.fuse_batch(_cache(False), K.FusionConfig(threshold=0.8, head_mode=head_mode))
    h = SHAPE["h"] if head_mode == "per_head" else 1
    assert got[0][0] == [0, 1, 2] and got[1][0] == [3, 4]
    assert got[0][1] + got[1][1] == [o.report.layer for o in full]
    r0 = next(x for x in got if x[2] is not None)
    before, after, per_rank, tables = r0[2:]
    assert before == sum(o.report.blocks_before for o in full)
    assert after == sum(o.report.blocks_after for o in full)
    assert per_rank == [sum(o.report.blocks_after for o in full[:3 * h]),
                        sum(o.report.blocks_after for o in full[3 * h:])]
    flat = [row for t in tables for row in t]
    assert flat == [o.fused.table.device_table.tolist() for o in full]


def test_layers_argument_matches_full_run():
    cache = _cache(False)
    full = K.fuse_batch(cache, K.FusionConfig(threshold=0.8))
    part = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), layers=range(2, 4))
    assert [o.report.layer for o in part] == [2, 3]
    for a, b in zip(part, full[2:4]):
        assert torch.equal(a.fused.table.device_table, b.fused.table.device_table)
        assert a.report.to_dict() == b.report.to_dict()
    with pytest.raises(K.ConfigError):
        K.fuse_batch(cache, K.FusionConfig(threshold=0.8), layers=[0, 2])
