"""Host-resident caches streamed to the GPU in layer chunks (defer_upload):
identical results to the device-resident path, NaN/Inf detection on device."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200 import fusion as F  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


@pytest.mark.parametrize("L", [3, 9])
@pytest.mark.parametrize("head_mode", ["folded", "per_head"])
def test_streamed_equals_resident(L, head_mode, monkeypatch):
    monkeypatch.setattr(F, "STREAM_LAYERS", 4)  # 9 layers -> chunks of 4, 4, 1
    B, p, t, h, d = 8, 16, 16, 2, 64
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=13)
    dims = K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L)
    cfg = K.FusionConfig(threshold=0.8, head_mode=head_mode)
    ref = K.fuse_batch(K.PagedKvCache(dims, Kt, Vt), cfg)
    host = K.PagedKvCache(dims, Kt.cpu().pin_memory(), Vt.cpu().pin_memory(), defer_upload=True)
    assert host.host_resident
    got = K.fuse_batch(host, cfg, in_place=True)
    assert not host.host_resident
    assert len(got) == len(ref)
    for a, b in zip(ref, got):
        assert a.report.layer == b.report.layer and a.report.head == b.report.head
        assert a.report.to_dict() == b.report.to_dict()
        np.testing.assert_array_equal(a.fused.table.device_table.cpu(), b.fused.table.device_table.cpu())
        assert a.fused.keys.phys_ids == b.fused.keys.phys_ids
        np.testing.assert_array_equal(a.fused.keys.directions, b.fused.keys.directions)
    # fused pool landed in the cache's device tensors (in_place)
    fused_ref = ref[0].fused.state.pool_k.view(host.keys_dev.shape)
    assert torch.equal(host.keys_dev.view(torch.int16), fused_ref.view(torch.int16))


def test_streamed_nan_raises():
    L, B, p, t, h, d = 2, 4, 8, 16, 2, 64
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1)
    Kh = Kt.cpu()
    Kh[1, 2, 3, 4, 1, 5] = float("nan")
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kh, Vt.cpu(), defer_upload=True)
    with pytest.raises(K.InvalidCacheError):
        K.fuse_batch(cache, K.FusionConfig(threshold=0.8))
