"""Pin the CPU oracle to the reference: every golden case recorded from the
reference implementation (tests/golden/make_golden.py) must be reproduced
exactly (integers / structure) and to 1e-12 (directions, sample moments)."""

import numpy as np
import pytest

import kvfuse_oracle as O
from conftest import golden, golden_cases, unit_inputs


def _check(case, res: O.OracleResult, arrays):
    name = case["name"]
    rep = case["report"]
    assert res.blocks_after == rep["blocks_after"]
    assert res.blocks_before == rep["blocks_before"]
    assert res.merge_calls == rep["merge_calls"]
    assert res.tree_depth == rep["tree_depth"]
    assert res.survivors == case["phys_ids"]
    np.testing.assert_array_equal(res.table, arrays[f"{name}/table"])
    np.testing.assert_array_equal(res.refcount, arrays[f"{name}/refcount"])
    # events: same order, same absorber / absorbed home slots
    ev = [[list(a), [list(s) for s in b]] for a, b in res.events]
    assert ev == rep["fused_events"]
    # fused directions of survivors
    ids = case["phys_ids"]
    np.testing.assert_allclose(res.kdir[ids], arrays[f"{name}/kdir"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(res.vdir[ids], arrays[f"{name}/vdir"], atol=1e-12, rtol=0)
    # per-merge records (post order)
    assert len(res.records) == len(case["records"])
    for got, want in zip(res.records, case["records"]):
        assert (got.level, got.left_blocks, got.right_blocks, got.fused_count, got.n) == (
            want["level"], want["left"], want["right"], want["fused"], want["n"])
        if got.n:
            assert got.s1 / got.n == pytest.approx(want["mean"], abs=1e-12)
            assert got.mn == pytest.approx(want["min"], abs=1e-12)
            assert got.mx == pytest.approx(want["max"], abs=1e-12)
    np.testing.assert_allclose(res.samples(), arrays[f"{name}/samples"], atol=1e-12, rtol=0)


@pytest.mark.parametrize(
    "case", golden_cases(("fast_fusion_fixture", "fast_fusion_rows", "hand")), ids=lambda c: c["name"]
)
def test_fast_fusion_cases(case):
    arrays, _ = golden()
    k, v, rows, bpr = unit_inputs(case)
    res = O.fuse_unit(k, v, rows, bpr, case["thr"])
    _check(case, res, arrays)


@pytest.mark.parametrize("case", golden_cases(("fuse_batch", "tree")), ids=lambda c: c["name"])
def test_fuse_batch_cases(case):
    arrays, _ = golden()
    if case["kind"] == "tree":
        K = arrays[f"tree/{case['B']}/keys"]
        V = arrays[f"tree/{case['B']}/values"]
        layer, gs = 0, None
    else:
        K = arrays[f"fixture/{case['fixture']}/keys"]
        V = arrays[f"fixture/{case['fixture']}/values"]
        layer, gs = case["layer"], case["group_size"]
    B, p = K.shape[1:3]
    res = O.fuse_unit(O.layer_unit(K, layer), O.layer_unit(V, layer), B, p, case["thr"],
                      O.bff_groups(B, gs))
    _check(case, res, arrays)


@pytest.mark.parametrize("case", golden_cases("fuse_chunks"), ids=lambda c: c["name"])
def test_fuse_chunks_cases(case):
    arrays, _ = golden()
    K = arrays[f"fixture/{case['fixture']}/keys"]
    V = arrays[f"fixture/{case['fixture']}/values"]
    L, B, p, t = K.shape[:4]
    C, bpc = O.cff_chunks(p, t, case["chunk_tokens"])
    res = O.fuse_unit(O.layer_unit(K, case["layer"]), O.layer_unit(V, case["layer"]), B * C, bpc,
                      case["thr"], O.cff_groups(B, C, None))
    _check(case, res, arrays)
    assert sorted(int(i) for i in np.nonzero(res.refcount > 1)[0]) == case["reusable"]


def test_refold_and_attention_golden():
    arrays, meta = golden()
    K = arrays["fixture/clusters4/keys"]
    V = arrays["fixture/clusters4/values"]
    B, p, t, h, d = K.shape[1:]
    res = O.fuse_unit(O.layer_unit(K, 0), O.layer_unit(V, 0), B, p, 0.91)
    kv, vv = O.refold(res, (t, h, d))
    np.testing.assert_allclose(kv, arrays["refold/clusters4/thr0.91/L0/keys"], atol=1e-12)
    np.testing.assert_allclose(vv, arrays["refold/clusters4/thr0.91/L0/values"], atol=1e-12)
    for a in meta["attention"]:
        q = arrays[f"att/{a['i']}/q"]
        out, s = O.paged_attention(q, kv, vv, a["row"], a["head"])
        np.testing.assert_allclose(out, arrays[f"att/{a['i']}/out_fused"], atol=1e-12)
        np.testing.assert_allclose(s, arrays[f"att/{a['i']}/probs_fused"], atol=1e-12)
        out_b, s_b = O.paged_attention(q, K[0], V[0], a["row"], a["head"])
        np.testing.assert_allclose(out_b, arrays[f"att/{a['i']}/out_base"], atol=1e-12)


def test_override_adopts_consistent_flip():
    # two blocks exactly at the threshold: the device may decide either way
    k = np.array([[1.0, 0.0], [np.cos(0.5), np.sin(0.5)]])
    thr = float(k[0] @ k[1] / np.linalg.norm(k[1]))
    base = O.fuse_unit(k, k, 2, 1, thr)
    assert base.blocks_after == 2
    forced = O.fuse_unit(k, k, 2, 1, thr, gpu_absorber=np.array([O.NONE, 0]), eps=1e-9)
    assert forced.blocks_after == 1 and forced.flips == 1 and forced.mismatches == 0
    bad = O.fuse_unit(k, k, 2, 1, thr - 0.1, gpu_absorber=np.array([O.NONE, O.NONE]), eps=1e-9)
    assert bad.mismatches == 1
