"""Host-side API of the drop-in (fusion.py:49-110, 126-202, 418-465): threshold
controller, configuration validation, report serialization. CPU tests mirror
the reference's test_fusion.py:240-360; the GPU tests replay acceptance 11
(tune_threshold) and the JSON / CSV / aggregate reports against the reference's
own outputs recorded in tests/golden (make_golden.py section 7)."""

import json

import numpy as np
import pytest

from conftest import golden

import paper_2601_03067_b200 as K
from paper_2601_03067_b200 import AdaptPolicy, ConfigError, FusionConfig, FusionReport, adapt_threshold
from paper_2601_03067_b200.errors import InsufficientDataError


def _report(samples, cr=1.0):
    blocks = 10
    return FusionReport(0, blocks, int(round(blocks / cr)), [], 1, 1,
                        np.asarray(samples, dtype=np.float64))


def test_adapt_policy_validation():
    with pytest.raises(ConfigError):
        AdaptPolicy(mode="nope", target=2.0, step=0.01, min_threshold=0.1, max_threshold=0.9)
    with pytest.raises(ConfigError):
        AdaptPolicy(mode="percentile", target=0.2, step=0.0, min_threshold=0.1, max_threshold=0.9)
    with pytest.raises(ConfigError):
        AdaptPolicy(mode="percentile", target=0.2, step=0.1, min_threshold=0.9, max_threshold=0.1)


@pytest.mark.parametrize("thr", [-1.0, 1.0, 1.5, -2.0])
def test_threshold_range(thr):
    with pytest.raises(ConfigError):
        FusionConfig(threshold=thr)


def test_config_validation():
    with pytest.raises(ConfigError):
        FusionConfig(threshold=0.5, variant="xff")
    with pytest.raises(ConfigError):
        FusionConfig(threshold=0.5, group_size=0)


def test_percentile_mode():
    pol = AdaptPolicy(mode="percentile", target=0.2, step=0.01, min_threshold=0.0, max_threshold=0.99)
    rep = _report(np.arange(1, 11) / 10.0)
    assert adapt_threshold(pol, rep, 0.5) == pytest.approx(0.82)  # 0.8-quantile, linear
    pol = AdaptPolicy(mode="percentile", target=0.2, step=0.01, min_threshold=0.0, max_threshold=0.5)
    assert adapt_threshold(pol, rep, 0.5) == 0.5
    with pytest.raises(InsufficientDataError):
        adapt_threshold(pol, _report([]), 0.5)


def test_target_compression_steps():
    pol = AdaptPolicy(mode="target-compression", target=2.0, step=0.01, min_threshold=0.1,
                      max_threshold=0.9)
    hi, lo = _report([0.5], cr=5.0), _report([0.5], cr=1.25)
    assert adapt_threshold(pol, hi, 0.5) == pytest.approx(0.51)
    assert adapt_threshold(pol, lo, 0.5) == pytest.approx(0.49)
    assert adapt_threshold(pol, hi, 0.9) == 0.9
    assert adapt_threshold(pol, lo, 0.1) == 0.1


def _clusters4():
    arrays, _ = golden()
    k = arrays["fixture/clusters4/keys"]
    v = arrays["fixture/clusters4/values"]
    L, B, p, t, h, d = k.shape
    return K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), k, v)


@pytest.mark.gpu
def test_tune_threshold_matches_reference():
    """Acceptance 11: same threshold trajectory and CRs as the reference."""
    want = golden()[1]["host"]["tune"]
    pol = AdaptPolicy(mode="target-compression", target=2.0, step=0.001, min_threshold=0.85,
                      max_threshold=0.97)
    thr, hist = K.tune_threshold(_clusters4(), FusionConfig(threshold=0.90), pol, rel_tol=0.1,
                                 max_iters=30)
    assert thr == want["final"]
    assert [list(h) for h in hist] == want["history"]
    with pytest.raises(ConfigError):
        K.tune_threshold(_clusters4(), FusionConfig(threshold=0.9),
                         AdaptPolicy(mode="percentile", target=0.2, step=0.01, min_threshold=0.1,
                                     max_threshold=0.9))


def _close(a, b):
    if isinstance(a, dict):
        assert a.keys() == b.keys()
        for k in a:
            _close(a[k], b[k])
    elif isinstance(a, list):
        assert len(a) == len(b)
        for x, y in zip(a, b):
            _close(x, y)
    elif isinstance(a, float) and isinstance(b, float):
        assert a == pytest.approx(b, abs=1e-12, rel=1e-12)
    else:
        assert a == b


@pytest.mark.gpu
def test_reports_json_csv_aggregate_match_reference():
    host = golden()[1]["host"]
    reports = [o.report for o in K.fuse_batch(_clusters4(), FusionConfig(threshold=0.91))]
    assert K.reports_to_csv(reports) == host["csv"]
    for r, want in zip(reports, host["json"]):
        _close(json.loads(r.to_json()), json.loads(want))
    _close(FusionReport.aggregate(reports).to_dict(), host["aggregate"])


@pytest.mark.gpu
def test_device_quantile_matches_numpy():
    import torch

    from paper_2601_03067_b200.fusion import device_quantile

    g = torch.Generator(device="cuda").manual_seed(3)
    for n, nan_frac in ((1, 0.0), (2, 0.0), (7, 0.3), (1000, 0.5), (100_003, 0.1)):
        x = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
        x[torch.rand(n, generator=g, device="cuda") < nan_frac] = float("nan")
        x[: n // 3] = torch.round(x[: n // 3] * 4) / 4  # ties
        if n > 1:
            x[0] = -0.0
        parts = [x[: n // 2], x[n // 2:]]
        h = x.cpu().numpy()
        h = h[~np.isnan(h)]
        for q in (0.0, 0.2, 0.5, 0.8, 0.93, 1.0):
            if h.size == 0:
                continue
            assert device_quantile(parts, q) == np.quantile(h, q), (n, q)
    with pytest.raises(InsufficientDataError):
        device_quantile([torch.full((5,), float("nan"), dtype=torch.float64, device="cuda")], 0.5)


@pytest.mark.gpu
def test_percentile_adaptation_on_device_samples():
    """Percentile mode over a fused cache's device samples equals the host path."""
    reports = [o.report for o in K.fuse_batch(_clusters4(), FusionConfig(threshold=0.91), keep_samples=True)]
    pol = AdaptPolicy(mode="percentile", target=0.2, step=0.01, min_threshold=0.0, max_threshold=0.99)
    agg = FusionReport.aggregate(reports)
    assert agg.device_samples() is not None
    dev = adapt_threshold(pol, agg, 0.5)
    for r in reports:
        r.similarity_samples  # materialise on the host -> host path
    host = adapt_threshold(pol, FusionReport.aggregate(reports), 0.5)
    want = float(np.quantile(np.concatenate([r.similarity_samples for r in reports]), 0.8))
    assert dev == host == want


def test_stream_chunks_cover_layers_in_order():
    """Host-resident streaming: layer chunks cover [0, L) in order, full STREAM_LAYERS
    chunks first, then halving so one layer's fusion is left after the last copy."""
    from paper_2601_03067_b200.fusion import STREAM_LAYERS, _stream_chunks

    for L in range(1, 70):
        ch = _stream_chunks(L)
        assert ch[0][0] == 0 and ch[-1][1] == L
        assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
        sizes = [c1 - c0 for c0, c1 in ch]
        assert all(0 < s <= STREAM_LAYERS for s in sizes)
        assert sizes == sorted(sizes, reverse=True)
        if L > 1:
            assert sizes[-1] == 1


def test_aggregate_events_lazy_and_equal():
    """FusionReport.aggregate concatenates the parts' events only when they are read, and
    they equal the reference's eager concatenation (fusion.py:158-171)."""
    from paper_2601_03067_b200.fusion import FusionEvent

    parts = [
        FusionReport(layer=i, blocks_before=8, blocks_after=8 - i, merge_calls=3, tree_depth=2,
                     fused_events=[FusionEvent((0, k), ((1, k),)) for k in range(i)],
                     similarity_samples=np.arange(i, dtype=np.float64))
        for i in range(4)
    ]
    agg = FusionReport.aggregate(parts)
    assert agg._events is None  # not built by aggregate itself
    assert agg.compression_ratio == 32 / (32 - 6) and agg.fused_blocks == 6
    assert agg._events is None  # CR and fused block count do not need the events
    assert agg.fused_events == [e for r in parts for e in r.fused_events]
    assert agg.merge_calls == 12 and agg.tree_depth == 2 and agg.layer == -1
    np.testing.assert_array_equal(agg.similarity_samples, np.concatenate([np.arange(i) for i in range(4)]))
    assert agg.to_dict()["fused_events"][0] == [[0, 0], [[1, 0]]]
