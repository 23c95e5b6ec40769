"""Tiny bf16 fusion runs (folded + per-head, tcgen05 path) for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_03067_b200 as K
from paper_2601_03067_b200.workload import synthetic_kv

for hm in ("folded", "per_head"):
    L, B, p, t, h, d = 1, 8, 64, 16, 8, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=5)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.8, head_mode=hm), keep_samples=True)
    torch.cuda.synchronize()
    print(hm, sum(o.report.blocks_before for o in outs) / sum(o.report.blocks_after for o in outs))
