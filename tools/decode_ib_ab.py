"""A/B of sharing-aware decode item sizes on one cfg4 layer (batch 256 x 8K), alternating
runs in one process so box-to-box noise cancels: python tools/decode_ib_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_03067_b200 as K
from paper_2601_03067_b200.workload import synthetic_kv

L, B, p, t, h, d, Hq = 1, 256, 512, 16, 8, 128, 32
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1)
cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
st = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), in_place=True, keep_samples=False)[0].fused.state
del Kt, Vt
q = torch.randn((B, Hq, d), device="cuda", dtype=torch.bfloat16)
ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
out = torch.empty((B, Hq, d), dtype=torch.float32, device="cuda")
lse = torch.empty((B, Hq), dtype=torch.float32, device="cuda")
scheds = {ib: K.state_decode_schedule(st, 0, B, p, item_blocks=ib) for ib in (8, 16)}


def run(ib, n=20):
    fn = lambda: K.paged_decode(q, st, 0, B, p, schedule=scheds[ib], out=out, lse=lse, workspace=ws)
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


res = {8: [], 16: []}
for _ in range(4):
    for ib in (16, 8):
        res[ib].append(run(ib))
for ib, v in res.items():
    print(f"IB={ib}: us/layer min {min(v):.1f} all {[round(x, 1) for x in v]}")
