"""Public API (fuse_batch on a device-resident cfg2 cache, in place) vs the bare engine run:
the host-side cost of the drop-in boundary (audit, report objects)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_03067_b200 as K  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

L, B, p, t, h, d = 32, 64, 256, 16, 8, 128
K0, V0 = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000)
Kw, Vw = torch.empty_like(K0), torch.empty_like(V0)
dims = K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L)
cfg = K.FusionConfig(threshold=0.8)
for audit in (True, False, True, False):
    times = []
    for _ in range(3):
        Kw.copy_(K0)
        Vw.copy_(V0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        outs = K.fuse_batch(K.PagedKvCache(dims, Kw, Vw), cfg, in_place=True, audit=audit)
        cr = sum(o.report.blocks_before for o in outs) / sum(o.report.blocks_after for o in outs)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
    print(f"fuse_batch(in_place, audit={audit}): {min(times):.1f} ms (wall, incl. report CR {cr:.4f})")
