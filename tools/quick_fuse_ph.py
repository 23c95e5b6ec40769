"""Per-head cfg2-shaped fusion of L layers, three runs (ncu target for the per-head tiles)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_03067_b200.engine import FusionEngine, Geometry  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B, p, t, h, d = 64, 256, 16, 8, 128
K0, V0 = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000)
geom = Geometry(L, B * p, t, h, d, 1)
eng = FusionEngine(geom, bff_plan(B, p, None), torch.bfloat16, "cuda")
for _ in range(3):
    st = eng.run(K0.clone().view(-1), V0.clone().view(-1), 0.8)
    torch.cuda.synchronize()
print("ok", int(st.live_count.sum()))
