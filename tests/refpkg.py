"""The installed reference package -- TEST INFRASTRUCTURE ONLY.

oracle/_ref is a pip --target install of /root/reference/pkg (unmodified,
git-ignored, shipped with the snapshot to the GPU box; __graft_entry__.build
creates it). Tests run it on the same bytes as the device path to pin parity
to the reference itself, not only to the oracle restatement.
"""

from __future__ import annotations

import sys
from pathlib import Path

REF = Path(__file__).resolve().parent.parent / "oracle" / "_ref"


def reference():
    if not (REF / "kvfuse").exists():
        raise RuntimeError(f"{REF} is missing: run __graft_entry__.build() where /root/reference exists")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import kvfuse

    return kvfuse


def reference_fuse(Kh, Vh, dims: dict, thr: float, variant: str = "bff", chunk_tokens=None,
                   group_size=None):
    """fuse_batch / fuse_chunks of the reference on float64 arrays (L, B, p, t, h, d),
    BLAS pinned to one thread (threaded BLAS is pathological here)."""
    reference()
    from kvfuse.core import CacheDims, PagedKvCache
    from kvfuse.fusion import FusionConfig, fuse_batch, fuse_chunks
    from threadpoolctl import threadpool_limits

    cache = PagedKvCache(CacheDims(**dims), Kh, Vh)
    with threadpool_limits(1):
        if variant == "cff":
            cfg = FusionConfig(threshold=thr, variant="cff", group_size=group_size)
            return fuse_chunks(cache, cfg, chunk_tokens)
        return fuse_batch(cache, FusionConfig(threshold=thr, group_size=group_size))
