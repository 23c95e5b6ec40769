"""Per-level similarity time of the library at $KVF_LIB (default: in-tree build)
on an 8-layer cfg2-shaped cache: A/B harness for sim kernel changes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_03067_b200 import _native as N
from paper_2601_03067_b200.engine import FusionEngine, Geometry
from paper_2601_03067_b200.schedule import bff_plan
from paper_2601_03067_b200.workload import synthetic_kv
L, B, p, t, h, d = 8, 64, 256, 16, 8, 128
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1)
geom = Geometry(L, B * p, t, h, d, 0)
plan = bff_plan(B, p, None)
eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device, N.PATH_TC)
best = None
for it in range(4):
    k, v = Kt.clone().reshape(-1), Vt.clone().reshape(-1)
    torch.cuda.synchronize()
    st = eng.run(k, v, 0.8, time_sim=True); torch.cuda.synchronize()
    sims = [a.elapsed_time(b) for a, b, _ in st.sim_events]
    if best is None or sum(sims) < sum(best): best = sims
tag = os.environ.get("KVF_LIB", "in-tree")
print(f"{tag}: sim {sum(best):.2f} ms {[round(x, 2) for x in best]} absorber_sum={int(st.absorber.long().sum())}", flush=True)
