"""Chunked-prefill attention over a CFF-fused context (kvf_chunk_prefill,
SURVEY §8f rank 2) vs a float64 reference on the refolded view: earlier
chunks fully visible, the chunk's own keys causal. Dedup (one Q K^T / P V per
physical block) and per-slot modes agree."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


def _reference(q, st, layer, B, p, chunk_blocks, chunk):
    g = st.geom
    L, NB, t, h, d = g.L, g.NB, g.t, g.h, g.d
    Tq = chunk_blocks * t
    Hq = q.shape[2]
    G = Hq // h
    pk = st.pool_k.view(L, NB, t, h, d)[layer].double()
    pv = st.pool_v.view(L, NB, t, h, d)[layer].double()
    tab = st.table[layer].long()
    ks = st.k_scale[layer].double()
    vs = st.v_scale[layer].double()
    Kl = (pk[tab] * ks[:, None, None, None]).view(B, p * t, h, d)
    Vl = (pv[tab] * vs[:, None, None, None]).view(B, p * t, h, d)
    nk = (chunk + 1) * Tq
    keys = torch.arange(nk, device=q.device)
    qi = torch.arange(Tq, device=q.device) + chunk * Tq
    mask = keys[None, :] > qi[:, None]  # causal in absolute token index
    out = torch.empty((B, Tq, Hq, d), dtype=torch.float64, device=q.device)
    for qh in range(Hq):
        kh = qh // G
        logits = torch.einsum("bqd,bkd->bqk", q[:, :, qh].double(), Kl[:, :nk, kh]) / math.sqrt(d)
        logits = logits.masked_fill(mask[None], float("-inf"))
        out[:, :, qh] = torch.einsum("bqk,bkd->bqd", torch.softmax(logits, -1), Vl[:, :nk, kh])
    return out


@pytest.mark.parametrize("G,d,path", [(4, 128, "mma"), (2, 64, "mma"), (8, 128, "mma"),
                                      (4, 128, "tc"), (8, 128, "tc"), (2, 128, "tc")])
def test_chunk_prefill_vs_reference(G, d, path):
    L, B, p, t, h = 1, 2, 64, 16, 2
    chunk_blocks = 16
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=81, variant="cff")
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    st = K.fuse_chunks(cache, K.FusionConfig(threshold=0.8, variant="cff"), chunk_blocks * t,
                       keep_samples=False)[0].fused.state
    assert int(st.live_count.sum()) < B * p
    torch.manual_seed(2)
    Hq = h * G
    for chunk in range(p // chunk_blocks):
        q = torch.randn((B, chunk_blocks * t, Hq, d), device="cuda", dtype=torch.bfloat16)
        want = _reference(q, st, 0, B, p, chunk_blocks, chunk)
        got = K.chunk_prefill(q, st, 0, B, p, chunk_blocks, chunk, path=path)
        torch.testing.assert_close(got.double(), want, atol=3e-3, rtol=3e-3)
        slot = K.chunk_prefill(q, st, 0, B, p, chunk_blocks, chunk, dedup=False, path=path)
        torch.testing.assert_close(got, slot, atol=2e-3, rtol=2e-3)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVF_RANDOM_CASES", "4"))))
def test_random_chunk_prefill_vs_reference(seed):
    """Seeded random CFF geometries (batch, chunk size, GQA group, kernel path) for
    chunked prefill with and without per-block reuse."""
    import numpy as np

    rng = np.random.default_rng(900 + seed)
    t, h, d = 16, 2, 128
    B = int(rng.integers(1, 4))
    chunk_blocks = int(rng.choice([8, 16]))
    C = int(rng.choice([2, 4]))
    p = chunk_blocks * C
    G = int(rng.choice([1, 2, 4, 8]))
    path = ["auto", "mma"][seed % 2]  # auto: tcgen05 where the shape allows
    Kt, Vt = synthetic_kv(1, B, p, t, h, d, dtype=torch.bfloat16, seed=950 + seed, variant="cff")
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=1), Kt, Vt)
    st = K.fuse_chunks(cache, K.FusionConfig(threshold=0.8, variant="cff"), chunk_blocks * t,
                       keep_samples=False)[0].fused.state
    g = torch.Generator(device="cuda").manual_seed(seed)
    for chunk in range(C):
        q = torch.randn((B, chunk_blocks * t, h * G, d), device="cuda", dtype=torch.bfloat16, generator=g)
        want = _reference(q, st, 0, B, p, chunk_blocks, chunk)
        for dedup in (True, False):
            got = K.chunk_prefill(q, st, 0, B, p, chunk_blocks, chunk, dedup=dedup, path=path)
            torch.testing.assert_close(got.double(), want, atol=3e-3, rtol=3e-3)
