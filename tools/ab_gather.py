"""A/B: staged vs gathered compaction on cfg2 (bench-like timing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_03067_b200.engine import FusionEngine, Geometry
from paper_2601_03067_b200.schedule import bff_plan
from paper_2601_03067_b200.workload import synthetic_kv
L, B, p, t, h, d = 32, 64, 256, 16, 8, 128
K0, V0 = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000)
Kw, Vw = torch.empty_like(K0), torch.empty_like(V0)
geom = Geometry(L, B * p, t, h, d, 0)
plan = bff_plan(B, p, None)
res = {}
for mode in ("staged", "gathered", "staged", "gathered"):
    eng = FusionEngine(geom, plan, torch.bfloat16, "cuda", compact_mode=mode)
    ts, sims = [], []
    for it in range(5):
        Kw.copy_(K0); Vw.copy_(V0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); st = eng.run(Kw.view(-1), Vw.view(-1), 0.8, time_sim=True); e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1))
            sims.append([a.elapsed_time(b) for a, b, _ in st.sim_events])
    res.setdefault(mode, []).append((sum(ts) / len(ts), [round(sum(x) / len(x), 2) for x in zip(*sims)]))
    live = int(st.live_count.sum())
    print(mode, f"step {sum(ts)/len(ts):.2f} ms", "sim per level", res[mode][-1][1], "live", live, flush=True)
    del eng
    torch.cuda.empty_cache()
