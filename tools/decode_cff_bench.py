"""Decode over a CFF-fused cache (blocks shared inside each request): unfused vs
request-major vs sharing-aware schedule with run dedup.

  python tools/decode_cff_bench.py [L B p]   (default: 2 layers, batch 64 x 16K, chunks of 2K)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_03067_b200 as K
from paper_2601_03067_b200.workload import synthetic_kv

L, B, p = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (2, 64, 1024)))
t, h, d, Hq = 16, 8, 128, 32
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=5, variant="cff")
K0, V0 = Kt.clone(), Vt.clone()
cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
outs = K.fuse_chunks(cache, K.FusionConfig(threshold=0.8, variant="cff"), 2048, in_place=True,
                     keep_samples=False)
st = outs[0].fused.state
cr = sum(o.report.blocks_before for o in outs) / sum(o.report.blocks_after for o in outs)
q = torch.randn((B, Hq, d), device="cuda", dtype=torch.bfloat16)
ident = torch.arange(B * p, dtype=torch.int32, device="cuda").repeat(L, 1)
ones = torch.ones((L, B * p), dtype=torch.float32, device="cuda")
unf = K.FusionState(st.geom, st.plan, 0.8, K0.view(-1), V0.view(-1), None, None, None, None, None,
                    None, None, ident, None, ones, ones)
scheds = [K.state_decode_schedule(st, l, B, p) for l in range(L)]
ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
out = torch.empty((B, Hq, d), dtype=torch.float32, device="cuda")
lse = torch.empty((B, Hq), dtype=torch.float32, device="cuda")


def timeit(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n / L


logical = 2 * B * p * t * h * d * 2
res = {
    "unfused": timeit(lambda: [K.paged_decode(q, unf, l, B, p, out=out, lse=lse, workspace=ws) for l in range(L)]),
    "fused_request_major": timeit(lambda: [K.paged_decode(q, st, l, B, p, out=out, lse=lse, workspace=ws) for l in range(L)]),
    "fused_sched": timeit(lambda: [K.paged_decode(q, st, l, B, p, schedule=scheds[l], out=out, lse=lse, workspace=ws) for l in range(L)]),
}
o1, _ = K.paged_decode(q, st, 0, B, p)
o2, _ = K.paged_decode(q, st, 0, B, p, schedule=scheds[0])
print(f"CFF L={L} B={B} ctx={p * t} CR={cr:.3f} repeats/layer={scheds[0].repeats} of {B * p} slots")
for k, v in res.items():
    print(f"  {k:20s} {v * 1e3:8.1f} us/layer  logical {logical / v / 1e6:7.0f} GB/s  tok/s(32 layers) {B / (v * 32 / 1e3):9.0f}")
print(f"  max |request-major - sched| = {(o1 - o2).abs().max().item():.2e}")
