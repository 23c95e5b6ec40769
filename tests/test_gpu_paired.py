"""Paired small merges (KVF_SIM_PAIRED): levels whose merge sides all fit one 128-row box run
two merges per tile on the diagonal of the CTA pair's 256 x 256 product (CTA c streams only
merge 2k + c's rows). Every similarity is the same chain of K16 MMAs on the same operand
rows, so decisions, pools and samples are bitwise those of one merge per tile; only the
per-warp moment slots regroup."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.engine import FusionEngine  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan, cff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


def _run(monkeypatch, paired, geom, plan, Kt, Vt, dtype, samples, **kw):
    monkeypatch.setenv("KVF_SIM_PAIRED", "1" if paired else "0")
    eng = FusionEngine(geom, plan, dtype, Kt.device, **kw)
    assert any(eng.paired) == paired
    st = eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8, keep_samples=samples)
    torch.cuda.synchronize()
    return st, eng


@pytest.mark.parametrize("case", ["cff", "bff_odd", "bff_f32_split", "bff_norms", "per_head", "group_size"])
@pytest.mark.parametrize("samples", [False, True], ids=["moments", "samples"])
def test_paired_matches_single(monkeypatch, case, samples):
    t, h, d = 16, 8, 128
    dtype = torch.float32 if case == "bff_f32_split" else torch.bfloat16
    kw = {}
    if case == "cff":  # 8 chunks of 128 blocks: level 1 = 4 merges of 128 x 128 per unit
        L, B, p = 2, 1, 1024
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=61, variant="cff")
        plan = cff_plan(B, 8, 128, None)
    elif case == "bff_odd":  # 6 rows: 3 level-1 merges per unit, the last tile half empty
        L, B, p = 2, 6, 64
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=62)
        plan = bff_plan(B, p, None)
    elif case == "bff_f32_split":  # cfg1-shaped: hi / lo operands and split-K
        L, B, p = 4, 8, 64
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=63)
        plan = bff_plan(B, p, None)
    elif case == "per_head":  # (layer, KV head) units: head-slice rows on paired tiles
        L, B, p = 2, 8, 64
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=65)
        plan = bff_plan(B, p, None)
    elif case == "group_size":  # independent trees of 3 rows (uneven merges inside a level)
        L, B, p = 2, 12, 96
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=66)
        plan = bff_plan(B, p, 3)
    else:  # fused level-1 key norms on paired tiles
        L, B, p = 8, 32, 128
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=64)
        plan = bff_plan(B, p, None)
        kw = dict(split=False)
    geom = K.Geometry(L, B * p, t, h, d, 1 if case == "per_head" else 0)
    a, ea = _run(monkeypatch, True, geom, plan, Kt, Vt, dtype, samples, **kw)
    b, eb = _run(monkeypatch, False, geom, plan, Kt, Vt, dtype, samples, **kw)
    split_any = max(ea.nsplit) > 1 or max(eb.nsplit) > 1
    if case == "bff_f32_split":
        assert split_any
    if case == "bff_norms":
        assert ea.fuse_knorm and eb.fuse_knorm and ea.paired[0]
    assert torch.equal(a.absorber, b.absorber)
    assert torch.equal(a.table, b.table) and torch.equal(a.refcount, b.refcount)
    bits = torch.int16 if dtype == torch.bfloat16 else torch.int32
    assert torch.equal(a.pool_k.view(bits), b.pool_k.view(bits))
    assert torch.equal(a.pool_v.view(bits), b.pool_v.view(bits))
    assert torch.equal(a.orig_knorm, b.orig_knorm)
    for sa, sb in zip(a.level_stats, b.level_stats):
        assert torch.equal(sa[..., :4], sb[..., :4])
        n = sa[..., 3:4].clamp(min=1)
        torch.testing.assert_close(sa[..., 4:6] / n, sb[..., 4:6] / n, rtol=0, atol=2e-5)
        torch.testing.assert_close(sa[..., 6:], sb[..., 6:], rtol=0, atol=3e-4 if split_any else 0)
    if samples:
        for xa, xb in zip(a.level_samples, b.level_samples):
            if split_any:  # split-K regroups the fp32 partial sums
                torch.testing.assert_close(torch.nan_to_num(xa), torch.nan_to_num(xb), rtol=0, atol=3e-4)
            else:
                assert torch.equal(xa.view(torch.int64), xb.view(torch.int64))
