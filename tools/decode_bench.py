"""Decode-only timing on a fused Llama-3-8B-shaped cache (batch 64 x 4K, 32 layers)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_03067_b200 as K
from paper_2601_03067_b200.attention import _decode
from paper_2601_03067_b200.workload import synthetic_kv
L = int(os.environ.get("L", "8"))
B, p, t, h, d = 64, 256, 16, 8, 128
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1)
cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
st = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), in_place=True, keep_samples=False)[0].fused.state
q = torch.randn((B, 32, d), device="cuda", dtype=torch.bfloat16)
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty((B, 32, d), device="cuda"); lse = torch.empty((B, 32), device="cuda")
def step():
    for layer in range(L):
        _decode(q, st.pool_k, st.pool_v, st.geom, layer, st.table, st.k_scale, st.v_scale, B, p, 32,
                d ** -0.5, out=out, lse=lse, workspace=ws)
step(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10 / L
print(f"tiles={os.environ.get('KVF_DECODE_TILES', 'default')} per-layer {ms*1e3:.1f} us  {2*B*p*t*h*d*2/ms/1e9:.0f} GB/s logical")
