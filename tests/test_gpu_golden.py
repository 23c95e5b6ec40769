"""GPU drop-in parity against the reference's own outputs (golden vectors
recorded from /root/reference by tests/golden/make_golden.py).

float64 caches run the float64 device path: tables, refcounts, survivors and
event lists must be identical; directions / sample moments within 1e-12."""

import numpy as np
import pytest

from conftest import golden, golden_cases, unit_inputs

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")


def _unfolded(x, rows, bpr):
    x = np.asarray(x, dtype=np.float64).reshape(rows, bpr, -1)
    n = np.linalg.norm(x, axis=-1)
    safe = np.where(n > 0, n, 1.0)
    return K.UnfoldedLayer(vectors=x / safe[..., None], norms=n)


def _check(case, oc, arrays, exact_dirs=1e-12):
    name = case["name"]
    rep = case["report"]
    got = oc.report.to_dict()
    for key in ("blocks_before", "blocks_after", "merge_calls", "tree_depth", "fused_events"):
        assert got[key] == rep[key], key
    assert got["compression_ratio"] == rep["compression_ratio"]
    sim, want = got["similarity"], rep["similarity"]
    assert sim["n"] == want["n"]
    for k in ("mean", "std", "min", "max"):
        if want[k] is None:
            assert sim[k] is None
        else:
            assert sim[k] == pytest.approx(want[k], abs=1e-12)
    assert list(oc.fused.keys.phys_ids) == case["phys_ids"]
    n = len(arrays[f"{name}/table"])
    bpr = oc.fused.key_norms.shape[1]
    tab = np.array([oc.table.entries[(s // bpr, s % bpr)] for s in range(n)])
    np.testing.assert_array_equal(tab, arrays[f"{name}/table"])
    ref = np.zeros(n, dtype=np.int64)
    for p_, c in oc.table.refcount.items():
        ref[p_] = c
    np.testing.assert_array_equal(ref, arrays[f"{name}/refcount"])
    np.testing.assert_allclose(oc.fused.keys.directions, arrays[f"{name}/kdir"], atol=exact_dirs, rtol=0)
    np.testing.assert_allclose(oc.fused.values.directions, arrays[f"{name}/vdir"], atol=exact_dirs, rtol=0)
    np.testing.assert_allclose(oc.report.similarity_samples, arrays[f"{name}/samples"], atol=1e-12, rtol=0)
    for m, w in zip(oc.report.merge_records, case["records"]):
        assert (m.level, m.left_blocks, m.right_blocks, m.fused_count, m.n_samples) == (
            w["level"], w["left"], w["right"], w["fused"], w["n"])
    oc.table.audit()


@pytest.mark.parametrize(
    "case", golden_cases(("fast_fusion_fixture", "fast_fusion_rows", "hand")), ids=lambda c: c["name"]
)
def test_fast_fusion_golden(case):
    arrays, _ = golden()
    k, v, rows, bpr = unit_inputs(case)
    oc = K.fast_fusion(_unfolded(k, rows, bpr), _unfolded(v, rows, bpr), thr=case["thr"])
    _check(case, oc, arrays)


def _fixture_cache(arrays, fx):
    k = arrays[f"fixture/{fx}/keys"]
    v = arrays[f"fixture/{fx}/values"]
    L, B, p, t, h, d = k.shape
    return K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), k, v)


def test_fuse_batch_golden():
    arrays, _ = golden()
    by = {}
    for c in golden_cases("fuse_batch"):
        by.setdefault((c["fixture"], c["thr"], c["group_size"]), []).append(c)
    for (fx, thr, gs), cases in by.items():
        cache = _fixture_cache(arrays, fx)
        outs = K.fuse_batch(cache, K.FusionConfig(threshold=thr, group_size=gs))
        for c in cases:
            _check(c, outs[c["layer"]], arrays)


@pytest.mark.parametrize("case", golden_cases("tree"), ids=lambda c: c["name"])
def test_tree_golden(case):
    arrays, _ = golden()
    k = arrays[f"tree/{case['B']}/keys"]
    v = arrays[f"tree/{case['B']}/values"]
    L, B, p, t, h, d = k.shape
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), k, v)
    oc = K.fuse_batch(cache, K.FusionConfig(threshold=case["thr"]))[0]
    _check(case, oc, arrays)


def test_fuse_chunks_golden():
    arrays, _ = golden()
    cache = _fixture_cache(arrays, "cff")
    for thr in (0.8, 0.9):
        outs = K.fuse_chunks(cache, K.FusionConfig(threshold=thr, variant="cff"), 32)
        for c in golden_cases("fuse_chunks"):
            if c["thr"] != thr:
                continue
            oc = outs[c["layer"]]
            _check(c, oc, arrays)
            assert sorted(oc.table.reusable) == c["reusable"]


def test_refold_and_attention_golden():
    arrays, meta = golden()
    cache = _fixture_cache(arrays, "clusters4")
    oc = K.fuse_batch(cache, K.FusionConfig(threshold=0.91))[0]
    view = K.refold(oc.fused)
    np.testing.assert_allclose(view.keys, arrays["refold/clusters4/thr0.91/L0/keys"], atol=1e-12)
    np.testing.assert_allclose(view.values, arrays["refold/clusters4/thr0.91/L0/values"], atol=1e-12)
    base = K.LayerView(keys=cache.keys[0], values=cache.values[0])
    for a in meta["attention"]:
        q = K.AttentionQuery(q=arrays[f"att/{a['i']}/q"], head=a["head"])
        out, s = K.paged_attention(q, view, a["row"])
        np.testing.assert_allclose(out, arrays[f"att/{a['i']}/out_fused"], atol=1e-12)
        np.testing.assert_allclose(s.probs, arrays[f"att/{a['i']}/probs_fused"], atol=1e-12)
        # straight through the fused table (no refold)
        out2, s2 = K.paged_attention(q, oc.fused, a["row"])
        np.testing.assert_allclose(out2, arrays[f"att/{a['i']}/out_fused"], atol=1e-12)
        out_b, s_b = K.paged_attention(q, base, a["row"])
        np.testing.assert_allclose(out_b, arrays[f"att/{a['i']}/out_base"], atol=1e-12)
        np.testing.assert_allclose(s_b.probs, arrays[f"att/{a['i']}/probs_base"], atol=1e-12)
