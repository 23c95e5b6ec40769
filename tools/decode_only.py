"""Fuse a small Llama-shaped cache, then run K6 decode repeatedly (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_03067_b200 as K
from paper_2601_03067_b200.workload import synthetic_kv
L, B, p, t, h, d = 2, 64, 256, 16, 8, 128
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1)
cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
st = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), in_place=True, keep_samples=False)[0].fused.state
q = torch.randn((B, 32, d), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    for layer in range(L):
        K.paged_decode(q, st, layer, B, p)
torch.cuda.synchronize()
print("ok")
