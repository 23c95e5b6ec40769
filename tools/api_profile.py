"""cProfile of repeated public fuse_batch calls on a device-resident cfg2 cache (host overhead)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_03067_b200 as K  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

L, B, p, t, h, d = 32, 64, 256, 16, 8, 128
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000)
cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
cfg = K.FusionConfig(threshold=0.8)


def once():
    outs = K.fuse_batch(cache, cfg)
    rep = K.FusionReport.aggregate([o.report for o in outs])
    return rep.compression_ratio


once()
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    cr = once()
    torch.cuda.synchronize()
    print(f"fuse_batch + aggregate: {(time.perf_counter() - t0) * 1e3:.1f} ms (CR {cr:.4f})")
pr = cProfile.Profile()
pr.enable()
once()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
