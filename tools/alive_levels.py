import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_03067_b200.engine import FusionEngine, Geometry
from paper_2601_03067_b200.schedule import bff_plan
from paper_2601_03067_b200.workload import synthetic_kv
L, B, p, t, h, d = 2, 64, 256, 16, 8, 128
K0, V0 = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000)
geom = Geometry(L, B * p, t, h, d, 0)
eng = FusionEngine(geom, bff_plan(B, p, None), torch.bfloat16, "cuda")
st = eng.run(K0.view(-1), V0.view(-1), 0.8)
for li, s in enumerate(st.level_stats):
    s = s[0].double().cpu()
    print(f"level {li+1}: merges {s.shape[0]} alive(left+right) {int((s[:,0]+s[:,1]).sum())} fused {int(s[:,2].sum())} pairs {float((s[:,0]*s[:,1]).sum()):.3e}")
