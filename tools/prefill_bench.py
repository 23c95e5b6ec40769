"""Chunked prefill over a CFF-fused cache: dedup vs per-slot (same kernel), and
flash-attn (library) over the unfused keys as a reference point.

  python tools/prefill_bench.py [B p chunk]   (default 4 requests x 16K, chunk 7 of 8 x 2K)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_03067_b200 as K
from paper_2601_03067_b200.workload import synthetic_kv

B, p, chunk = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (4, 1024, 7)))
L, t, h, d, Hq, cb = 1, 16, 8, 128, 32, 128
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=5, variant="cff")
K0, V0 = Kt.clone(), Vt.clone()
cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
st = K.fuse_chunks(cache, K.FusionConfig(threshold=0.8, variant="cff"), cb * t, in_place=True,
                   keep_samples=False)[0].fused.state
Tq = cb * t
q = torch.randn((B, Tq, Hq, d), device="cuda", dtype=torch.bfloat16)
order = K.state_decode_schedule(st, 0, B, p).order[0]
prev = chunk * cb
tab = st.table[0].view(B, p)[:, :prev]
uniq = sum(len(torch.unique(r)) for r in tab)


def timeit(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


out = torch.empty((B, Tq, Hq, d), dtype=torch.float32, device="cuda")
PATH = os.environ.get("PATH_KIND", "auto")
t_dedup = timeit(lambda: K.chunk_prefill(q, st, 0, B, p, cb, chunk, order=order, dedup=True, out=out, path=PATH))
t_slot = timeit(lambda: K.chunk_prefill(q, st, 0, B, p, cb, chunk, order=order, dedup=False, out=out, path=PATH))
a = K.chunk_prefill(q, st, 0, B, p, cb, chunk, order=order, dedup=True, path=PATH)
b = K.chunk_prefill(q, st, 0, B, p, cb, chunk, order=order, dedup=False, path=PATH)
tk = (chunk + 1) * Tq
flops = 4.0 * B * Hq * Tq * (prev * t + Tq / 2) * d  # causal dense attention FLOPs
line = (f"path={PATH} B={B} ctx={p * t} chunk={chunk} earlier slots {B * prev} -> unique blocks {uniq} "
        f"(x{B * prev / uniq:.2f}); dense-equivalent {flops / 1e9:.0f} GFLOP\n"
        f"  chunk_prefill dedup    {t_dedup:7.3f} ms  ({flops / t_dedup / 1e9:6.0f} TFLOP/s dense-equivalent)\n"
        f"  chunk_prefill per-slot {t_slot:7.3f} ms  ({flops / t_slot / 1e9:6.0f} TFLOP/s)  speedup x{t_slot / t_dedup:.2f}"
        f"  max|diff| {(a - b).abs().max().item():.2e}")
try:
    from flash_attn import flash_attn_func

    kf = K0[0].view(B, p * t, h, d)[:, :tk]
    vf = V0[0].view(B, p * t, h, d)[:, :tk]
    t_fa = timeit(lambda: flash_attn_func(q, kf, vf, causal=True))
    line += f"\n  flash-attn (library) over the unfused keys {t_fa:7.3f} ms ({flops / t_fa / 1e9:6.0f} TFLOP/s)"
except Exception as exc:  # library optional
    line += f"\n  flash-attn unavailable: {str(exc)[:100]}"
print(line)
