"""Chunked level statistics (few, large merges: C CTAs per merge) against the one-CTA
path. Member segments are sorted after an atomic fill, so every merge sums its members
in the same ascending order: decisions, tables, refcounts and fused pools are bitwise
equal; MergeRecord counters are exact; the similarity moments are regrouped float64 sums
of the same tile partials."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.engine import FusionEngine  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan, cff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


def _run(monkeypatch, chunked, geom, plan, Kt, Vt, dtype):
    monkeypatch.setenv("KVF_LS_CHUNKED", "1" if chunked else "0")
    eng = FusionEngine(geom, plan, dtype, Kt.device)
    st = eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8)
    torch.cuda.synchronize()
    return st


@pytest.mark.parametrize("case", ["bff", "cff", "per_head", "f32"])
def test_chunked_level_stats_match(monkeypatch, case):
    t, h, d = 16, 8, 128
    dtype = torch.float32 if case == "f32" else torch.bfloat16
    if case == "cff":
        L, B, p = 2, 2, 512
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=41, variant="cff")
        plan = cff_plan(B, 4, 128, None)
    else:
        L, B, p = 2, 16, 128
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=40)
        plan = bff_plan(B, p, None)
    geom = K.Geometry(L, B * p, t, h, d, 1 if case == "per_head" else 0)
    a = _run(monkeypatch, True, geom, plan, Kt, Vt, dtype)
    b = _run(monkeypatch, False, geom, plan, Kt, Vt, dtype)
    assert torch.equal(a.absorber, b.absorber)
    assert torch.equal(a.table, b.table) and torch.equal(a.refcount, b.refcount)
    bits = torch.int16 if dtype == torch.bfloat16 else torch.int32
    assert torch.equal(a.pool_k.view(bits), b.pool_k.view(bits))
    assert torch.equal(a.pool_v.view(bits), b.pool_v.view(bits))
    assert torch.equal(a.k_scale, b.k_scale) and torch.equal(a.v_scale, b.v_scale)
    for sa, sb in zip(a.level_stats, b.level_stats):
        assert torch.equal(sa[..., :4], sb[..., :4])  # left / right / fused / sample counts
        torch.testing.assert_close(sa[..., 4:6], sb[..., 4:6], rtol=1e-12, atol=1e-9)
        assert torch.equal(sa[..., 6:], sb[..., 6:])  # min / max


def test_chunked_level_stats_deterministic(monkeypatch):
    L, B, p, t, h, d = 1, 32, 256, 16, 8, 128  # 8,192 blocks: the top merges take the chunked path
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=42)
    geom = K.Geometry(L, B * p, t, h, d, 0)
    plan = bff_plan(B, p, None)
    monkeypatch.delenv("KVF_LS_CHUNKED", raising=False)
    eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device)
    runs = [eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8) for _ in range(3)]
    for st in runs[1:]:
        assert torch.equal(st.pool_k.view(torch.int16), runs[0].pool_k.view(torch.int16))
        for sa, sb in zip(st.level_stats, runs[0].level_stats):
            assert torch.equal(sa, sb)
