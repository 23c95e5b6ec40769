"""K6 paged decode over fused caches vs a float64 torch reference that
materialises the logical view through the block table (refold semantics,
core.py:285-305) and applies exact softmax attention (attention.py:58-80),
with GQA and ragged sequence lengths."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.attention import _decode  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


def _reference(q, st, layer, B, p, seq_blocks=None):
    g = st.geom
    L, NB, t, h, d = g.L, g.NB, g.t, g.h, g.d
    pk = st.pool_k.view(L, NB, t, h, d)[layer].double()
    pv = st.pool_v.view(L, NB, t, h, d)[layer].double()
    Hq = q.shape[1]
    G = Hq // h
    out = torch.empty((B, Hq, d), dtype=torch.float64, device=q.device)
    for kvh in range(h):
        u = layer * h + kvh if g.head_mode else layer
        tab = st.table[u].long()
        ks = st.k_scale[u].double()
        vs = st.v_scale[u].double()
        Kl = (pk[tab][:, :, kvh, :] * ks[:, None, None]).view(B, p * t, d)
        Vl = (pv[tab][:, :, kvh, :] * vs[:, None, None]).view(B, p * t, d)
        for gg in range(G):
            qh = kvh * G + gg
            logits = torch.einsum("btd,bd->bt", Kl, q[:, qh].double()) / math.sqrt(d)
            if seq_blocks is not None:
                n = (seq_blocks.long() * t)[:, None]
                mask = torch.arange(p * t, device=q.device)[None, :] >= n
                logits = logits.masked_fill(mask, float("-inf"))
            w = torch.softmax(logits, dim=1)
            out[:, qh] = torch.einsum("bt,btd->bd", w, Vl)
    return out


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
@pytest.mark.parametrize("d,G,head_mode", [(128, 4, "folded"), (64, 2, "per_head"), (128, 1, "folded")])
def test_decode_vs_reference(dtype, d, G, head_mode):
    L, B, p, t, h = 2, 6, 40, 16, 4
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=31)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.8, head_mode=head_mode), keep_samples=False)
    st = outs[0].fused.state
    assert sum(o.report.blocks_after for o in outs) < sum(o.report.blocks_before for o in outs)
    torch.manual_seed(0)
    q = torch.randn((B, h * G, d), device="cuda", dtype=dtype)
    seq = torch.tensor([p, p - 3, 1, 17, p, 5], dtype=torch.int32, device="cuda")
    for layer in range(L):
        for sb in (None, seq):
            got, lse = K.paged_decode(q, st, layer, B, p, seq_blocks=sb)
            want = _reference(q, st, layer, B, p, sb)
            tol = 2e-3 if dtype == torch.bfloat16 else 1e-4
            torch.testing.assert_close(got.double(), want, atol=tol, rtol=tol)
            assert torch.isfinite(lse).all()


def test_decode_unfused_matches_fused_when_nothing_fuses():
    """Orthogonal blocks never fuse: the fused state decodes exactly like the raw cache."""
    L, B, p, t, h, d = 1, 4, 8, 16, 2, 128
    gen = torch.Generator(device="cuda").manual_seed(5)
    Kt = torch.randn((L, B, p, t, h, d), device="cuda", generator=gen).bfloat16()
    Vt = torch.randn((L, B, p, t, h, d), device="cuda", generator=gen).bfloat16()
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    st = K.fuse_batch(cache, K.FusionConfig(threshold=0.99))[0].fused.state
    assert int(st.live_count.sum()) == B * p
    q = torch.randn((B, 2 * h, d), device="cuda", dtype=torch.bfloat16)
    got, _ = K.paged_decode(q, st, 0, B, p)
    want = _reference(q, st, 0, B, p)
    torch.testing.assert_close(got.double(), want, atol=2e-3, rtol=2e-3)


@pytest.mark.parametrize("ib", [8, 16])
@pytest.mark.parametrize("d,G,head_mode", [(128, 4, "folded"), (64, 2, "per_head"), (128, 8, "folded")])
def test_scheduled_decode_vs_reference(d, G, head_mode, ib):
    """Sharing-aware schedule: same attention as the request-major reference."""
    L, B, p, t, h = 2, 7, 45, 16, 4
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=37)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.8, head_mode=head_mode), keep_samples=False)
    st = outs[0].fused.state
    torch.manual_seed(1)
    q = torch.randn((B, h * G, d), device="cuda", dtype=torch.bfloat16)
    seq = torch.tensor([p, p - 3, 1, 17, p, 5, 9], dtype=torch.int32, device="cuda")
    nit = (p + ib - 1) // ib
    for layer in range(L):
        for sb in (None, seq):
            sched = K.state_decode_schedule(st, layer, B, p, seq_blocks=sb, item_blocks=ib)
            nh = h if head_mode == "per_head" else 1
            nblk = (sb.long() if sb is not None else torch.full((B,), p, device="cuda")).cpu()
            n_valid = int(sum((int(n) + ib - 1) // ib for n in nblk))
            assert sched.n_items.cpu().tolist() == [n_valid] * nh
            for hu in range(nh):
                u = layer * h + hu if head_mode == "per_head" else layer
                tab, ksc, vsc = st.table[u].cpu(), st.k_scale[u].cpu(), st.v_scale[u].cpu()
                valid_slots = torch.cat([b * p + torch.arange(int(nblk[b])) for b in range(B)])
                refs = torch.bincount(tab[valid_slots].long(), minlength=tab.numel())
                meta = sched.meta[hu, :n_valid].cpu().long()
                phys = sched.phys[hu, :n_valid].cpu()
                # items swept by the physical block of their middle slot
                nvalid = (phys >= 0).sum(1)
                keys = [int(phys[i, (int(nvalid[i]) - 1) // 2]) for i in range(len(phys))]
                assert keys == sorted(keys)
                assert sorted(meta.tolist()) == sorted(
                    b * nit + k for b in range(B) for k in range((int(nblk[b]) + ib - 1) // ib))
                for row, it in enumerate(meta.tolist()):
                    b, k = divmod(it, nit)
                    pos = sched.order[hu, b, k * ib:(k + 1) * ib].cpu().long()
                    pos = pos[(torch.arange(len(pos)) + k * ib) < int(nblk[b])]
                    n = len(pos)
                    assert (phys[row, n:] == -1).all()
                    slots = b * p + pos
                    assert torch.equal(phys[row, :n], tab[slots])
                    # K scale magnitudes; the sign bit flags blocks that no other valid slot
                    # of the unit references (the decode's L2 evict-first hint)
                    ks_row = sched.ks[hu, row, :n].cpu()
                    assert torch.equal(ks_row.abs(), ksc[slots])
                    assert torch.equal(torch.signbit(ks_row), refs[tab[slots].long()] == 1)
                    assert torch.equal(sched.vs[hu, row, :n].cpu(), vsc[slots])
                for b in range(B):
                    n = int(nblk[b])
                    o = sched.order[hu, b, :n].cpu().long()
                    assert sorted(o.tolist()) == list(range(n))
                    assert (sched.order[hu, b, n:] == -1).all()
                    ph = tab[b * p + o]
                    assert (ph[1:] >= ph[:-1]).all()
            got, lse = K.paged_decode(q, st, layer, B, p, schedule=sched)
            want = _reference(q, st, layer, B, p, sb)
            torch.testing.assert_close(got.double(), want, atol=2e-3, rtol=2e-3)
            plain, lse0 = K.paged_decode(q, st, layer, B, p, seq_blocks=sb)
            torch.testing.assert_close(got, plain, atol=1e-3, rtol=1e-3)
            torch.testing.assert_close(lse, lse0, atol=1e-3, rtol=1e-3)


def test_scheduled_decode_many_sharers():
    """A batch where most slots point at a few shared blocks (high refcount)."""
    L, B, p, t, h, d = 1, 32, 24, 16, 2, 128
    gen = torch.Generator(device="cuda").manual_seed(9)
    base_k = torch.randn((4, t, h, d), device="cuda", generator=gen)
    base_v = torch.randn((4, t, h, d), device="cuda", generator=gen)
    pick = torch.randint(0, 4, (B, p), device="cuda", generator=gen)
    noise = 0.02
    Kt = (base_k[pick] + noise * torch.randn((B, p, t, h, d), device="cuda", generator=gen))[None].bfloat16()
    Vt = (base_v[pick] + noise * torch.randn((B, p, t, h, d), device="cuda", generator=gen))[None].bfloat16()
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    st = K.fuse_batch(cache, K.FusionConfig(threshold=0.9), keep_samples=False)[0].fused.state
    assert int(st.live_count.sum()) < B * p // 8
    q = torch.randn((B, 4 * h, d), device="cuda", dtype=torch.bfloat16)
    sched = K.state_decode_schedule(st, 0, B, p)
    got, _ = K.paged_decode(q, st, 0, B, p, schedule=sched)
    want = _reference(q, st, 0, B, p)
    torch.testing.assert_close(got.double(), want, atol=2e-3, rtol=2e-3)


@pytest.mark.parametrize("ib", [8, 16])
def test_scheduled_decode_cff_repeats(ib):
    """CFF shares blocks inside a request: a request's context holds the same
    fused block several times (runs in the sorted slot order). Runs are loaded
    and multiplied once; the result must equal the slot-by-slot reference."""
    L, B, p, t, h, d = 1, 6, 64, 16, 4, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=53, variant="cff")
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    outs = K.fuse_chunks(cache, K.FusionConfig(threshold=0.8, variant="cff"), 4 * t, keep_samples=False)
    st = outs[0].fused.state
    tab = st.table[0].view(B, p)
    repeats = sum(int(len(r) - len(torch.unique(r))) for r in tab)
    assert repeats > B * p // 4  # CFF: many in-request repeats
    q = torch.randn((B, 4 * h, d), device="cuda", dtype=torch.bfloat16)
    seq = torch.tensor([p, 63, 1, 40, 17, p], dtype=torch.int32, device="cuda")
    for sb in (None, seq):
        sched = K.state_decode_schedule(st, 0, B, p, seq_blocks=sb, item_blocks=ib)
        got, lse = K.paged_decode(q, st, 0, B, p, schedule=sched)
        want = _reference(q, st, 0, B, p, sb)
        torch.testing.assert_close(got.double(), want, atol=2e-3, rtol=2e-3)
        plain, lse0 = K.paged_decode(q, st, 0, B, p, seq_blocks=sb)
        torch.testing.assert_close(lse, lse0, atol=1e-3, rtol=1e-3)


@pytest.mark.parametrize("t,d", [(32, 128), (32, 64), (16, 64)])
def test_scheduled_decode_block_sizes(t, d):
    """32-token blocks (6-warp variant) and d = 64 through the scheduled path."""
    L, B, p, h = 1, 5, 24, 2
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=71)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    st = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), keep_samples=False)[0].fused.state
    q = torch.randn((B, 3 * h, d), device="cuda", dtype=torch.bfloat16)
    seq = torch.tensor([p, 3, 24, 11, 1], dtype=torch.int32, device="cuda")
    for sb in (None, seq):
        sched = K.state_decode_schedule(st, 0, B, p, seq_blocks=sb)
        got, _ = K.paged_decode(q, st, 0, B, p, schedule=sched)
        want = _reference(q, st, 0, B, p, sb)
        torch.testing.assert_close(got.double(), want, atol=2e-3, rtol=2e-3)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVF_RANDOM_CASES", "6"))))
def test_random_decode_vs_reference(seed):
    """Seeded random shapes through both decode paths (request-major and sharing-aware,
    with and without ragged lengths) against the float64 refold + softmax reference."""
    rng = np.random.default_rng(500 + seed)
    B = int(rng.integers(1, 10))
    p = int(rng.integers(1, 70))
    h = int(rng.choice([1, 2, 4, 8]))
    G = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([64, 128]))
    t = 16
    head_mode = ["folded", "per_head"][seed % 2]
    Kt, Vt = synthetic_kv(1, B, p, t, h, d, dtype=torch.bfloat16, seed=600 + seed)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=1), Kt, Vt)
    st = K.fuse_batch(cache, K.FusionConfig(threshold=float(rng.choice([0.7, 0.8])), head_mode=head_mode),
                      keep_samples=False)[0].fused.state
    q = torch.randn((B, h * G, d), device="cuda", dtype=torch.bfloat16,
                    generator=torch.Generator(device="cuda").manual_seed(seed))
    seq = torch.tensor(rng.integers(1, p + 1, size=B), dtype=torch.int32, device="cuda")
    for sb in (None, seq):
        want = _reference(q, st, 0, B, p, sb)
        got, _ = K.paged_decode(q, st, 0, B, p, seq_blocks=sb)
        torch.testing.assert_close(got.double(), want, atol=2e-3, rtol=2e-3)
        sched = K.state_decode_schedule(st, 0, B, p, seq_blocks=sb)
        got2, _ = K.paged_decode(q, st, 0, B, p, schedule=sched)
        torch.testing.assert_close(got2.double(), want, atol=2e-3, rtol=2e-3)
