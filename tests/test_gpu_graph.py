"""A fusion run captured as one CUDA graph replays to exactly the eager result
(same launches, same buffers), including the persistent similarity kernel's
tile scheduler state across replays."""

import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200.engine import FusionEngine  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan, cff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


@pytest.mark.parametrize("variant", ["bff", "cff"])
def test_graph_replay_equals_eager(variant):
    L, B, p, t, h, d = 2, 4, 64, 16, 8, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=77, variant=variant)
    geom = K.Geometry(L, B * p, t, h, d, 0)
    plan = bff_plan(B, p, None) if variant == "bff" else cff_plan(B, 4, p // 4, None)
    eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device)
    ref = eng.run(Kt.clone().view(-1), Vt.clone().view(-1), 0.8)
    ref = {k: getattr(ref, k).clone() for k in ("absorber", "table", "refcount", "k_scale", "live_count")}
    Kw, Vw = Kt.clone(), Vt.clone()
    cap = eng.capture(Kw.view(-1), Vw.view(-1), 0.8)
    for _ in range(3):  # restore the pristine pool, replay
        Kw.copy_(Kt)
        Vw.copy_(Vt)
        st = cap.replay()
        torch.cuda.synchronize()
        for k, v in ref.items():
            assert torch.equal(getattr(st, k), v), k
    assert int(st.live_count.sum()) < L * B * p
