"""Compacted levels in unit chunks (staging budget): running the top levels
unit-chunk by unit-chunk must give bitwise the same decisions, pools and statistics
as one launch over all units."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200 import engine as E  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


@pytest.mark.parametrize("head_mode", [0, 1])
def test_unit_chunks_bitwise(head_mode, monkeypatch):
    L, B, p, t, h, d = 5, 16, 32, 16, 2, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=29)
    geom = K.Geometry(L, B * p, t, h, d, head_mode)
    plan = bff_plan(B, p, None)
    states = []
    for budget in (1 << 40, 2 * B * p * geom.r * 2):  # everything at once / 2 units per chunk
        monkeypatch.setenv("KVF_STAGE_BUDGET", repr(budget / 2**30))  # GiB
        eng = E.FusionEngine(geom, plan, torch.bfloat16, Kt.device, compact_from=2, split=False)
        assert eng.stage_units == (geom.units if budget > 1 << 39 else 2)
        states.append(eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8, keep_samples=True))
    a, b = states
    assert torch.equal(a.absorber, b.absorber) and torch.equal(a.table, b.table)
    assert torch.equal(a.pool_k.view(torch.int16), b.pool_k.view(torch.int16))
    for sa, sb in zip(a.level_stats, b.level_stats):
        assert torch.equal(sa, sb)
    for xa, xb in zip(a.level_samples, b.level_samples):
        assert torch.equal(xa.view(torch.int64), xb.view(torch.int64))
    assert a.inexact_pairs() == b.inexact_pairs() == 0
