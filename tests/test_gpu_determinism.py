"""Bitwise determinism under repetition: 100 CUDA-graph replays of
one fusion step (bf16 exact mode with compaction, float32 hi/lo split with split-K)
from the same pristine pool must reproduce tables, absorbers, fused pools, shadow
rows, similarity moments and scales bit for bit -- every reduction in the path is
fixed-order (first-match by atomicMin of ids, split-K partials summed in split
order, level statistics reduced per warp slot in fixed order)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.engine import FusionEngine  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

REPLAYS = 100


def _snapshot(st):
    out = [st.absorber.clone(), st.table.clone(), st.refcount.clone(), st.live_count.clone(),
           st.pool_k.clone(), st.pool_v.clone(), st.k_scale.clone(), st.v_scale.clone()]
    out += [s.clone() for s in st.level_stats]
    return out


@pytest.mark.parametrize("dtype,shape", [
    (torch.bfloat16, (2, 16, 32, 16, 8, 128)),  # 4 levels: compaction of the top ones
    (torch.float32, (2, 8, 64, 16, 8, 128)),    # split operands + split-K
], ids=["bf16-exact", "f32-splitk"])
def test_graph_replays_bitwise(dtype, shape):
    L, B, p, t, h, d = shape
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=23)
    eng = FusionEngine(K.Geometry(L, B * p, t, h, d, 0), bff_plan(B, p, None), dtype, Kt.device)
    if dtype == torch.float32:
        assert max(eng.nsplit) > 1
    else:
        assert eng.exact and eng.compact_from is not None
    Kw, Vw = Kt.clone(), Vt.clone()
    g = eng.capture(Kw.view(-1), Vw.view(-1), 0.8)
    ref = None
    for i in range(REPLAYS):
        Kw.copy_(Kt)
        Vw.copy_(Vt)
        st = g.replay()
        snap = _snapshot(st)
        if eng.shadow is not None:  # rows are taken in arrival order: compare them per block
            idx = eng.sidx.flatten()
            snap.append(eng.shadow[idx[idx >= 0].long()].clone())
            snap.append((idx >= 0).clone())
        if ref is None:
            ref = snap
            continue
        for a, b in zip(snap, ref):
            assert torch.equal(a.view(torch.uint8), b.view(torch.uint8)), f"replay {i} differs"
