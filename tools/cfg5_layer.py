"""One layer of BASELINE configs[4] (Llama-3-70B KV: batch 256 x 16K, 8 KV heads,
d = 128, bf16): fuse it on one GPU, time it, audit the table.

  python tools/cfg5_layer.py [group_size|none] [layers]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_03067_b200.engine import FusionEngine, Geometry, audit
from paper_2601_03067_b200.schedule import bff_plan
from paper_2601_03067_b200.workload import synthetic_kv

gs = None if len(sys.argv) < 2 or sys.argv[1] == "none" else int(sys.argv[1])
L = int(sys.argv[2]) if len(sys.argv) > 2 else 1
B, p, t, h, d = 256, 1024, 16, 8, 128
t0 = time.time()
plan = bff_plan(B, p, gs)
print(f"plan {time.time() - t0:.2f}s depth {plan.tree_depth}", flush=True)
geom = Geometry(1, B * p, t, h, d, 0)
eng = FusionEngine(geom, plan, torch.bfloat16, "cuda")
print(f"engine ready {time.time() - t0:.2f}s, mem {torch.cuda.memory_allocated() / 1e9:.1f} GB", flush=True)
for layer in range(L):
    K, V = synthetic_kv(1, B, p, t, h, d, dtype=torch.bfloat16, seed=500 + layer)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = eng.run(K.view(-1), V.view(-1), 0.8, time_sim=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    sims = [a.elapsed_time(b) for a, b, _ in st.sim_events]
    flops = sum(float((2 * s[..., 0].double() * s[..., 1].double()).sum()) for s in st.level_stats) * geom.r
    ok = audit(st.table, st.refcount, st.alive, 1, geom.NB)
    cr = geom.NB / int(st.live_count.sum())
    print(f"layer {layer}: {ms:.1f} ms (sim {sum(sims):.1f} ms, {flops / sum(sims) / 1e9:.0f} TFLOP/s, "
          f"{flops / 1e12:.1f} TFLOP) CR {cr:.3f} audit {ok} KV GB/s {2 * K.numel() * 2 / ms / 1e6:.0f} "
          f"mem peak {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
    del K, V, st
