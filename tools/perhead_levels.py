"""Per-level similarity times, folded vs per-head units, same cache (4 layers of cfg2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_03067_b200.engine import FusionEngine, Geometry
from paper_2601_03067_b200.schedule import bff_plan
from paper_2601_03067_b200.workload import synthetic_kv
L, B, p, t, h, d = 4, 64, 256, 16, 8, 128
K0, V0 = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000)
plan = bff_plan(B, p, None)
for hm in (0, 1, 0, 1):
    geom = Geometry(L, B * p, t, h, d, hm)
    eng = FusionEngine(geom, plan, torch.bfloat16, "cuda", compact_from=None if len(sys.argv) > 1 else "auto")
    for it in range(3):
        Kw, Vw = K0.clone(), V0.clone()
        st = eng.run(Kw.view(-1), Vw.view(-1), 0.8, time_sim=True)
        torch.cuda.synchronize()
    sims = [a.elapsed_time(b) for a, b, _ in st.sim_events]
    fl = [float((2 * s[..., 0].double() * s[..., 1].double()).sum()) * geom.r for s in st.level_stats]
    print("per_head" if hm else "folded  ", " ".join(f"{x:6.2f}ms/{f / x / 1e9:5.0f}TF" for x, f in zip(sims, fl)), flush=True)
