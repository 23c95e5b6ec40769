import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_03067_b200 import _native as N, schedule
from paper_2601_03067_b200.engine import FusionEngine, Geometry
from paper_2601_03067_b200.schedule import bff_plan
from paper_2601_03067_b200.workload import synthetic_kv
L, B, p, t, h, d = 8, 64, 256, 16, 8, 128
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1)
geom = Geometry(L, B * p, t, h, d, 0)
ref = None
for band in (1, 4, 8, 16, 1000):
    schedule.TILE_BAND = band
    plan = bff_plan(B, p, None)
    for lv in plan.levels:
        lv.tiling.__func__.__defaults__ = (band,)
    eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device, N.PATH_TC)
    best = None
    for it in range(3):
        k, v = Kt.clone().reshape(-1), Vt.clone().reshape(-1)
        torch.cuda.synchronize()
        st = eng.run(k, v, 0.8, time_sim=True); torch.cuda.synchronize()
        sims = [a.elapsed_time(b) for a, b, _ in st.sim_events]
        if best is None or sum(sims) < sum(best): best = sims
    if ref is None: ref = st.absorber.clone()
    print(f"band={band} sim {sum(best):.2f} ms {[round(x, 2) for x in best]} same={torch.equal(ref, st.absorber)}", flush=True)
