"""Wall time of the public fuse_chunks on a device-resident cfg3 cache (CFF, 32 layers x 16K)
and of per-layer report access, vs the device step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_03067_b200 as K  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

L, B, p, t, h, d = 32, 1, 1024, 16, 8, 128
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000, variant="cff")
cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
cfg = K.FusionConfig(threshold=0.8, variant="cff")
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outs = K.fuse_chunks(cache, cfg, 2048)
    cr = K.FusionReport.aggregate([o.report for o in outs]).compression_ratio
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    js = [o.report.to_json() for o in outs]
    t2 = time.perf_counter()
    print(f"fuse_chunks + aggregate CR {cr:.4f}: {(t1 - t0) * 1e3:.1f} ms; per-layer to_json x32: {(t2 - t1) * 1e3:.1f} ms")
