"""Wide similarity tile (KVF_PATH_TC_WIDE): a CTA pair computes 512 x 256 similarities
per tile (256 A rows per CTA, both TMEM halves holding one accumulator) instead of
256 x 256 with a double-buffered accumulator. Each similarity is the same chain of
K16 tcgen05 MMAs over the same operands, so decisions, tables, refcounts, fused
pools and every sample must be identical to the narrow tile; only the per-warp
moment slots regroup (fp32 sums in another order)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.engine import FusionEngine  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan, cff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


def _engine(monkeypatch, wide, geom, plan, dtype, device, **kw):
    monkeypatch.setenv("KVF_SIM_WIDE", "1" if wide else "0")
    monkeypatch.setenv("KVF_SIM_PAIRED", "0")  # every level on the tile under test
    return FusionEngine(geom, plan, dtype, device, split=False, **kw)


def _compare(a, b, samples):
    assert torch.equal(a.absorber, b.absorber)
    assert torch.equal(a.table, b.table) and torch.equal(a.refcount, b.refcount)
    assert torch.equal(a.alive, b.alive)
    bits = torch.int16 if a.pool_k.dtype == torch.bfloat16 else torch.int32
    assert torch.equal(a.pool_k.view(bits), b.pool_k.view(bits))
    assert torch.equal(a.pool_v.view(bits), b.pool_v.view(bits))
    for sa, sb in zip(a.level_stats, b.level_stats):
        assert torch.equal(sa[..., :4], sb[..., :4])  # counts
        n = sa[..., 3:4].clamp(min=1)
        torch.testing.assert_close(sa[..., 4:6] / n, sb[..., 4:6] / n, rtol=0, atol=1e-5)
        assert torch.equal(sa[..., 6:], sb[..., 6:])  # min / max: single samples
    if samples:
        for xa, xb in zip(a.level_samples, b.level_samples):
            assert torch.equal(xa.view(torch.int64), xb.view(torch.int64))


@pytest.mark.parametrize("samples", [False, True], ids=["moments", "samples"])
@pytest.mark.parametrize("compact", ["auto", None], ids=["staged", "direct"])
def test_wide_matches_narrow_bff(monkeypatch, samples, compact):
    L, B, p, t, h, d = 2, 16, 96, 16, 8, 128  # 1,536 blocks per layer: ragged 512-row tiles
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=31)
    geom = K.Geometry(L, B * p, t, h, d, 0)
    plan = bff_plan(B, p, None)
    states = []
    for wide in (True, False):
        eng = _engine(monkeypatch, wide, geom, plan, torch.bfloat16, Kt.device, compact_from=compact)
        assert all(eng.wide) == wide
        if compact == "auto":
            assert eng.compact_from is not None
        states.append(eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8,
                              keep_samples=samples))
    _compare(*states, samples)


def test_wide_matches_narrow_float32_and_cff(monkeypatch):
    # float32 pool: three hi / lo passes per tile on the wide tile too
    L, B, p, t, h, d = 2, 8, 64, 16, 8, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.float32, seed=32)
    geom = K.Geometry(L, B * p, t, h, d, 0)
    plan = bff_plan(B, p, None)
    st = [_engine(monkeypatch, w, geom, plan, torch.float32, Kt.device).run(
        Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8, keep_samples=True) for w in (True, False)]
    _compare(*st, True)
    # CFF chunk tree (unequal merge sizes inside a level)
    L, B, p = 2, 1, 768
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=33, variant="cff")
    geom = K.Geometry(L, B * p, t, h, d, 0)
    plan = cff_plan(B, 6, 128, None)
    st = [_engine(monkeypatch, w, geom, plan, torch.bfloat16, Kt.device).run(
        Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8, keep_samples=True) for w in (True, False)]
    _compare(*st, True)


def test_wide_auto_selection(monkeypatch):
    """auto: the wide tile only where every merge's left side fills it and the level has
    at least two waves of tiles; never with split-K, per-head units or gathered rows."""
    monkeypatch.delenv("KVF_SIM_WIDE", raising=False)
    dev = torch.device("cuda", 0)
    L, B, p, t, h, d = 8, 64, 256, 16, 8, 128  # cfg2 layer geometry (no pool needed)
    geom = K.Geometry(L, B * p, t, h, d, 0)
    eng = FusionEngine(geom, bff_plan(B, p, None), torch.bfloat16, dev)
    assert eng.wide == [False, True, True, True, True, True]
    eng = FusionEngine(K.Geometry(L, B * p, t, h, d, 1), bff_plan(B, p, None), torch.bfloat16, dev)
    assert not any(eng.wide)
