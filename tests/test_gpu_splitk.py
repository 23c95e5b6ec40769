"""Split-K similarity (tcgen05 path): levels with few, long-K tiles -- BASELINE
configs[0] (cfg1) and CFF chunk trees -- split each tile's k-steps over several
CTA pairs and sum the fp32 partials in split order. Decisions (exact mode and
float64 re-scores) and therefore tables, refcounts and events must be identical
to the unsplit kernel; similarity moments agree to fp32 summation order."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.engine import FusionEngine, choose_split  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan, cff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


def test_choose_split_model():
    assert choose_split(16, 256, 74) == 4  # cfg1 level 1: 16 tiles -> 64 items
    assert choose_split(200, 256, 74) == 1  # enough tiles already
    assert choose_split(64, 256, 74) == 1  # more than half a wave (cfg3 level 2)
    assert choose_split(16, 32, 74) == 1  # short K (per-head units): never split
    assert choose_split(1, 768, 74) == 8  # capped at SPLIT_MAX (serial fix-up of the partials)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
@pytest.mark.parametrize("variant", ["bff", "cff"])
def test_splitk_matches_unsplit(dtype, variant):
    if variant == "bff":
        L, B, p, t, h, d = 4, 8, 64, 16, 8, 128  # cfg1 shape
        plan = bff_plan(B, p, None)
    else:
        L, B, p, t, h, d = 1, 1, 256, 16, 8, 128  # CFF: 8 chunks of 32 blocks, few tiles
        plan = cff_plan(B, 8, 32, None)
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=17, variant=variant)
    geom = K.Geometry(L, B * p, t, h, d, 0)
    states = []
    for split in (True, False):
        eng = FusionEngine(geom, plan, dtype, Kt.device, split=split)
        assert (max(eng.nsplit) > 1) == split
        states.append(eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8, keep_samples=True))
    a, b = states
    assert torch.equal(a.absorber, b.absorber)
    assert torch.equal(a.table, b.table) and torch.equal(a.refcount, b.refcount)
    assert torch.equal(a.pool_k.view(torch.int16 if dtype == torch.bfloat16 else torch.int32),
                       b.pool_k.view(torch.int16 if dtype == torch.bfloat16 else torch.int32))
    for sa, sb in zip(a.level_stats, b.level_stats):
        assert torch.equal(sa[..., :4], sb[..., :4])  # counts
        n = sa[..., 3:4].clamp(min=1)  # moments per sample: fp32 sums regroup across splits
        torch.testing.assert_close(sa[..., 4:6] / n, sb[..., 4:6] / n, rtol=0, atol=2e-5)
        # min / max: single samples, each within the tensor-core accumulation error (~1e-4)
        torch.testing.assert_close(sa[..., 6:], sb[..., 6:], rtol=0, atol=3e-4)
    for xa, xb in zip(a.level_samples, b.level_samples):
        assert torch.equal(xa.isnan(), xb.isnan())
        torch.testing.assert_close(torch.nan_to_num(xa), torch.nan_to_num(xb), rtol=0, atol=3e-4)


def test_splitk_bitwise_deterministic():
    L, B, p, t, h, d = 4, 8, 64, 16, 8, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=18)
    eng = FusionEngine(K.Geometry(L, B * p, t, h, d, 0), bff_plan(B, p, None), torch.bfloat16, Kt.device)
    assert max(eng.nsplit) > 1
    runs = [eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8, keep_samples=True) for _ in range(5)]
    for st in runs[1:]:
        assert torch.equal(st.absorber, runs[0].absorber)
        for xa, xb in zip(st.level_samples, runs[0].level_samples):
            assert torch.equal(xa.view(torch.int64), xb.view(torch.int64))
