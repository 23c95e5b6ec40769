"""Per-level profile of a cfg2-shaped fusion run: alive rows, fused counts, similarity time.

usage: python tools/level_profile.py [L] [compact_from] [B] [p]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_03067_b200 import _native as N  # noqa: E402
from paper_2601_03067_b200.engine import FusionEngine, Geometry  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cf = sys.argv[2] if len(sys.argv) > 2 else "auto"
cf = None if cf == "none" else ("auto" if cf == "auto" else int(cf))
B = int(sys.argv[3]) if len(sys.argv) > 3 else 64
p = int(sys.argv[4]) if len(sys.argv) > 4 else 256
t, h, d = 16, 8, 128
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000)
geom = Geometry(L, B * p, t, h, d, 0)
plan = bff_plan(B, p, None)
eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device, N.PATH_TC, compact_from=cf)
for it in range(3):
    k, v = Kt.clone().reshape(-1), Vt.clone().reshape(-1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = eng.run(k, v, 0.8, time_sim=True)
    e1.record()
    torch.cuda.synchronize()
print(f"L={L} compact_from={eng.compact_from} total {e0.elapsed_time(e1):.2f} ms")
for li, ((a, b, _), s) in enumerate(zip(st.sim_events, st.level_stats)):
    s = s.double()
    nl, nr, nf = s[..., 0].sum().item(), s[..., 1].sum().item(), s[..., 2].sum().item()
    fl = float((2 * s[..., 0] * s[..., 1]).sum().item()) * geom.r
    ms = a.elapsed_time(b)
    lvl = plan.levels[li]
    print(f"level {li} height {lvl.height} merges/unit {s.shape[1]} left_alive {nl:.0f} right_alive {nr:.0f} "
          f"fused {nf:.0f} ({nf / max(nr, 1):.3f} of right) sim {ms:.2f} ms {fl / ms / 1e9:.0f} TFLOP/s")
