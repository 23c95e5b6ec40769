"""Key norms fused into the level-1 similarity launch (KVF_SIM_WRITE_NORMS): the norm
warps read every operand row from the shared-memory ring after the MMAs, so the K pass
of kvf_block_norms disappears. The 8-element fp32 partials are the standalone kernel's;
only their float64 summation order differs, so the float32 norms agree to one ulp (and
in practice bitwise), and decisions, tables, pools and statistics are identical."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.engine import FusionEngine  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan, cff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


def _run(monkeypatch, fused, geom, plan, Kt, Vt, **kw):
    monkeypatch.setenv("KVF_FUSE_KNORM", "1" if fused else "0")
    eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device, split=False, **kw)  # split-K: separate pass
    assert eng.fuse_knorm == fused
    st = eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8, keep_samples=True)
    torch.cuda.synchronize()
    return st


@pytest.mark.parametrize("case", ["bff", "bff_ragged", "cff", "zero_blocks", "per_head"])
def test_fused_knorm_matches_separate_pass(monkeypatch, case):
    t, h, d = 16, 8, 128
    if case == "cff":
        L, B, p = 2, 2, 512
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, seed=51, variant="cff")
        plan = cff_plan(B, 4, 128, None)
    else:
        L, B, p = 2, 16, (100 if case == "bff_ragged" else 128)
        Kt, Vt = synthetic_kv(L, B, p, t, h, d, seed=50)
        plan = bff_plan(B, p, None)
    if case == "zero_blocks":  # not fusable: key norm 0 (fusion.py:218)
        Kt[:, 3, 7] = 0
        Kt[:, 11, 0] = 0
    geom = K.Geometry(L, B * p, t, h, d, 1 if case == "per_head" else 0)
    a = _run(monkeypatch, True, geom, plan, Kt, Vt)
    b = _run(monkeypatch, False, geom, plan, Kt, Vt)
    rel = ((a.orig_knorm - b.orig_knorm).abs() / b.orig_knorm.clamp(min=1e-30)).max().item()
    assert rel <= 2.0**-23
    assert torch.equal(a.fusable, b.fusable)
    if case == "zero_blocks":
        assert int((a.fusable == 0).sum()) == 2 * L
    assert torch.equal(a.orig_knorm, b.orig_knorm)  # same partials, exact float64 sums
    assert torch.equal(a.absorber, b.absorber)
    assert torch.equal(a.table, b.table) and torch.equal(a.refcount, b.refcount)
    assert torch.equal(a.pool_k.view(torch.int16), b.pool_k.view(torch.int16))
    assert torch.equal(a.pool_v.view(torch.int16), b.pool_v.view(torch.int16))
    for sa, sb in zip(a.level_stats, b.level_stats):
        assert torch.equal(sa[..., :4], sb[..., :4])
        torch.testing.assert_close(sa[..., 4:], sb[..., 4:], rtol=1e-6, atol=1e-6)
    for xa, xb in zip(a.level_samples, b.level_samples):
        torch.testing.assert_close(torch.nan_to_num(xa), torch.nan_to_num(xb), rtol=0, atol=1e-6)


def test_fused_knorm_selection(monkeypatch):
    monkeypatch.delenv("KVF_FUSE_KNORM", raising=False)
    dev = torch.device("cuda", 0)
    g = K.Geometry(4, 64 * 256, 16, 8, 128, 0)
    assert FusionEngine(g, bff_plan(64, 256, None), torch.bfloat16, dev).fuse_knorm  # cfg2 shape
    # a row outside every level-1 merge (odd batch), float32 pools: separate pass
    assert not FusionEngine(K.Geometry(1, 5 * 64, 16, 8, 128, 0), bff_plan(5, 64, None),
                            torch.bfloat16, dev).fuse_knorm
    assert not FusionEngine(K.Geometry(1, 16 * 64, 16, 8, 128, 0), bff_plan(16, 64, None),
                            torch.float32, dev).fuse_knorm
    # level-1 merges wider than one tile (1,024 blocks per request, cfg5 shape)
    assert not FusionEngine(K.Geometry(1, 4 * 1024, 16, 8, 128, 0), bff_plan(4, 1024, None),
                            torch.bfloat16, dev).fuse_knorm
