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
