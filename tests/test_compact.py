"""Compacted fused layers: KVFF v2 serialization round
trips and format errors, rank-to-rank transfer over gloo (CPU, world 2), and
-- on the GPU -- compaction of a fused state against its paged pool, with
decode over the compact pool equal to decode over the paged pool."""

import multiprocessing as mp
import socket

import pytest
import torch

from paper_2601_03067_b200.compact import CompactLayer, load_fused, save_fused
from paper_2601_03067_b200.errors import FormatError


def _layer(seed, n_live=5, B=2, p=4, shape=(4, 2, 8), dtype=torch.bfloat16, layer=0):
    g = torch.Generator().manual_seed(seed)
    keys = torch.randn((n_live, *shape), generator=g).to(dtype)
    values = torch.randn((n_live, *shape), generator=g).to(dtype)
    phys = torch.sort(torch.randperm(B * p, generator=g)[:n_live]).values.int()
    table = torch.randint(0, n_live, (B * p,), generator=g, dtype=torch.int32)
    ks = torch.rand(B * p, generator=g) + 0.5
    vs = torch.rand(B * p, generator=g) + 0.5
    return CompactLayer(layer, B, p, keys, values, phys, table, ks, vs)


def _equal(a, b):
    assert (a.layer, a.B, a.p_blocks, a.block_shape) == (b.layer, b.B, b.p_blocks, b.block_shape)
    for x, y in ((a.keys, b.keys), (a.values, b.values), (a.phys_ids, b.phys_ids), (a.table, b.table),
                 (a.k_scale, b.k_scale), (a.v_scale, b.v_scale)):
        assert x.dtype == y.dtype and torch.equal(x.cpu(), y.cpu())


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_kvff2_round_trip(tmp_path, dtype):
    layers = [_layer(s, n_live=3 + s, dtype=dtype, layer=s) for s in range(3)]
    path = tmp_path / "f.kvff"
    n = save_fused(path, layers)
    assert n == path.stat().st_size
    back = load_fused(path)
    assert len(back) == 3
    for a, b in zip(layers, back):
        _equal(a, b)


def test_kvff2_errors(tmp_path):
    path = tmp_path / "f.kvff"
    save_fused(path, [_layer(1)])
    data = path.read_bytes()
    bad = tmp_path / "bad.kvff"
    bad.write_bytes(b"XXXX" + data[4:])
    with pytest.raises(FormatError, match="magic"):
        load_fused(bad)
    bad.write_bytes(data[:4] + (1).to_bytes(4, "little") + data[8:])
    with pytest.raises(FormatError, match="version"):
        load_fused(bad)
    bad.write_bytes(data[:-3])
    with pytest.raises(FormatError, match="truncated"):
        load_fused(bad)
    bad.write_bytes(data + b"\0")
    with pytest.raises(FormatError, match="trailing"):
        load_fused(bad)
    bad.write_bytes(data[:10])
    with pytest.raises(FormatError, match="too short"):
        load_fused(bad)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2601_03067_b200.compact import recv_layer, send_layer

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        if rank == 0:  # the "prefill" rank ships two fused layers
            for s in (3, 4):
                send_layer(_layer(s, n_live=4 + s, layer=s), dst=1)
        else:
            got = [recv_layer(0, "cpu") for _ in range(2)]
            for s, cl in zip((3, 4), got):
                _equal(_layer(s, n_live=4 + s, layer=s), cl)
            q.put("ok")
    finally:
        dist.destroy_process_group()


def test_send_recv_layers_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) == "ok"


@pytest.mark.gpu
def test_compact_fused_state_gpu(tmp_path):
    import paper_2601_03067_b200 as K
    from paper_2601_03067_b200.compact import compact_cache, compact_decode_schedule, decode_compact
    from paper_2601_03067_b200.workload import synthetic_kv

    L, B, p, t, h, d = 2, 8, 40, 16, 4, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=61)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    st = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), keep_samples=False)[0].fused.state
    layers = compact_cache(st, B, p)
    pk = st.pool_k.view(L, B * p, t, h, d)
    pv = st.pool_v.view(L, B * p, t, h, d)
    q = torch.randn((B, 4 * h, d), device="cuda", dtype=torch.bfloat16)
    for cl in layers:
        u = cl.layer
        assert cl.n_live == int(st.live_count[u]) < B * p
        assert torch.equal(cl.phys_ids, st.live_ids[u, :cl.n_live])
        assert torch.equal(cl.keys, pk[u][cl.phys_ids.long()])
        assert torch.equal(cl.values, pv[u][cl.phys_ids.long()])
        # slot s reads the same block through the dense table
        assert torch.equal(cl.phys_ids[cl.table.long()], st.table[u])
        sched_c = compact_decode_schedule(cl)
        sched_p = K.state_decode_schedule(st, u, B, p)
        a, la = decode_compact(q, cl, sched_c)
        b, lb = K.paged_decode(q, st, u, B, p, schedule=sched_p)
        assert torch.equal(a, b) and torch.equal(la, lb)  # same items, same order, same data
    path = tmp_path / "fused.kvff"
    save_fused(path, layers)
    back = load_fused(path, device="cuda")
    for a, b in zip(layers, back):
        _equal(a, b)
