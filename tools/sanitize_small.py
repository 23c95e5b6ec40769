"""Tiny runs of every kernel family for compute-sanitizer (memcheck / synccheck /
racecheck / initcheck): bf16 folded + per-head fusion (exact mode, tcgen05),
float32 fusion (hi/lo split operands + split-K), CFF, request-major and
scheduled decode, chunked prefill."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_03067_b200 as K
from paper_2601_03067_b200.workload import synthetic_kv

torch.cuda.set_device(0)
for hm in ("folded", "per_head"):
    L, B, p, t, h, d = 1, 8, 64, 16, 8, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=5)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.8, head_mode=hm), keep_samples=True)
    torch.cuda.synchronize()
    print("bf16", hm, sum(o.report.blocks_before for o in outs) / sum(o.report.blocks_after for o in outs))
# wide similarity tiles (512 x 256 per CTA pair) + chunked level statistics, staged compaction
os.environ["KVF_SIM_WIDE"] = "1"
os.environ["KVF_LS_CHUNKED"] = "1"
for dt in (torch.bfloat16, torch.float32):
    Kt, Vt = synthetic_kv(2, 16, 96, 16, 8, 128, dtype=dt, seed=10)
    cache = K.PagedKvCache(K.CacheDims(B=16, p=96, t=16, h=8, d=128, L=2), Kt, Vt)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), keep_samples=dt == torch.float32)
    torch.cuda.synchronize()
    print("wide + chunked stats", dt, outs[0].report.compression_ratio)
del os.environ["KVF_SIM_WIDE"], os.environ["KVF_LS_CHUNKED"]
# paired level-1 merges with the key norms fused into the launch (no split-K)
from paper_2601_03067_b200.engine import FusionEngine, Geometry  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402
Kt, Vt = synthetic_kv(2, 16, 64, 16, 8, 128, dtype=torch.bfloat16, seed=12)
eng = FusionEngine(Geometry(2, 16 * 64, 16, 8, 128, 0), bff_plan(16, 64, None), torch.bfloat16, Kt.device,
                   split=False)
assert eng.paired[0] and eng.fuse_knorm
st = eng.run(Kt.reshape(-1).clone(), Vt.reshape(-1).clone(), 0.8, keep_samples=True)
torch.cuda.synchronize()
print("paired + fused norms", int(st.live_count.sum()))
# compacted levels with the alive rows gathered from the pool (cp.async + peer relay)
from paper_2601_03067_b200 import _native as N  # noqa: E402
from paper_2601_03067_b200.engine import FusionEngine, Geometry  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402

Kt, Vt = synthetic_kv(1, 16, 64, 16, 8, 128, dtype=torch.bfloat16, seed=9)
eng = FusionEngine(Geometry(1, 16 * 64, 16, 8, 128, 0), bff_plan(16, 64, None), torch.bfloat16, Kt.device,
                   N.PATH_TC, compact_from=2, compact_mode="gathered")
st = eng.run(Kt.reshape(-1).clone(), Vt.reshape(-1).clone(), 0.8)
torch.cuda.synchronize()
print("gathered", int(st.live_count.sum()))
# float32: split operands, split-K (few long tiles)
Kt, Vt = synthetic_kv(2, 8, 64, 16, 8, 128, dtype=torch.float32, seed=6)
cache = K.PagedKvCache(K.CacheDims(B=8, p=64, t=16, h=8, d=128, L=2), Kt, Vt)
outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.8))
print("f32", outs[0].fused.state.path_name, outs[0].report.compression_ratio)
# CFF + chunked prefill over the fused context
Kt, Vt = synthetic_kv(1, 2, 64, 16, 2, 128, dtype=torch.bfloat16, seed=7, variant="cff")
cache = K.PagedKvCache(K.CacheDims(B=2, p=64, t=16, h=2, d=128, L=1), Kt, Vt)
oc = K.fuse_chunks(cache, K.FusionConfig(threshold=0.8, variant="cff"), 256)[0]
st = oc.fused.state
q = torch.randn(2, 16 * 16, 8, 128, device="cuda", dtype=torch.bfloat16)
try:
    K.chunk_prefill(q, st, 0, 2, 64, 16, 3)
except Exception as exc:  # shape limits of the prefill kernels are not the point here
    print("prefill skipped:", str(exc)[:80])
# decode: request-major and sharing-aware
Kt, Vt = synthetic_kv(1, 16, 64, 16, 2, 128, dtype=torch.bfloat16, seed=8)
cache = K.PagedKvCache(K.CacheDims(B=16, p=64, t=16, h=2, d=128, L=1), Kt, Vt)
st = K.fuse_batch(cache, K.FusionConfig(threshold=0.8))[0].fused.state
qd = torch.randn(16, 8, 128, device="cuda", dtype=torch.bfloat16)
o1, _ = K.paged_decode(qd, st, 0, 16, 64)
o2, _ = K.paged_decode(qd, st, 0, 16, 64, schedule=K.state_decode_schedule(st, 0, 16, 64))
torch.cuda.synchronize()
print("decode max diff", float((o1 - o2).abs().max()))
