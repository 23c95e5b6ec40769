"""Exact-decision parity (north star "bit-exact except pairs within a
stated epsilon"): the device path against the float64 oracle with a 1e-9
exemption band -- no near-threshold slack -- and against the installed
reference package (oracle/_ref, the unmodified kvfuse) on identical inputs,
including BASELINE configs[0] (cfg1: 4 layers x 8 requests x 1024 tokens, 8 KV
heads, d = 128, fp32) at full shape.

bf16 pools run in exact mode (fp32 shadow rows of the fused key directions,
kern_exact.cu); float32 pools run the tcgen05 path on the hi/lo bf16 split with
float64 re-scores of the band. Flips are counted by the oracle and must be 0;
any pair decided differently outside the 1e-9 band is a mismatch."""

import numpy as np
import pytest
import torch

import kvfuse_oracle as O

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200 import _native as N  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

from refpkg import reference_fuse  # noqa: E402

EPS_EXACT = 1e-9
MAX_FLIPS = 0  # a flip needs |sim_ref - thr| <= 1e-9: none expected at these sizes


def _cache(L, B, p, t, h, d, dtype, seed, variant="bff"):
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=dtype, seed=seed, variant=variant)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    return cache, Kt.double().cpu().numpy(), Vt.double().cpu().numpy()


def _check_exact(outs, Kh, Vh, rows, bpr, thr, groups=None, per_head=False):
    flips = exempt = 0
    for oc in outs:
        st = oc.fused.state
        u = oc.fused.unit
        assert st.exact
        assert st.inexact_pairs() == 0 and st.inexact_blocks() == 0
        head = oc.fused.head if per_head else None
        ref = O.fuse_unit(O.layer_unit(Kh, oc.report.layer, head), O.layer_unit(Vh, oc.report.layer, head),
                          rows, bpr, thr, groups, gpu_absorber=st.absorber[u].cpu().numpy(),
                          eps=EPS_EXACT, keep_samples=False)
        assert ref.mismatches == 0, ref.mismatch_detail
        np.testing.assert_array_equal(st.table[u].cpu().numpy(), ref.table)
        np.testing.assert_array_equal(st.refcount[u].cpu().numpy(), ref.refcount)
        assert oc.report.blocks_after == ref.blocks_after
        ev = [[list(a), [list(s) for s in b]] for a, b in ref.events]
        assert oc.report.to_dict()["fused_events"] == ev
        flips += ref.flips
        exempt += ref.exempt_pairs
    assert flips <= MAX_FLIPS, f"{flips} flips within {EPS_EXACT} of the threshold"
    return flips, exempt


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
@pytest.mark.parametrize("head_mode", ["folded", "per_head"])
@pytest.mark.parametrize("thr", [0.8, 0.7])
def test_exact_bff_vs_oracle(dtype, head_mode, thr):
    L, B, p, t, h, d = 2, 8, 24, 16, 2, 128
    cache, Kh, Vh = _cache(L, B, p, t, h, d, dtype, seed=31)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=thr, head_mode=head_mode), keep_samples=False)
    assert outs[0].fused.state.geom.head_mode == (head_mode == "per_head")
    _check_exact(outs, Kh, Vh, B, p, thr, per_head=head_mode == "per_head")


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_exact_cff_vs_oracle(dtype):
    L, B, p, t, h, d = 2, 3, 64, 16, 2, 128
    chunk = 8 * t  # C = 8 chunks of 8 blocks
    cache, Kh, Vh = _cache(L, B, p, t, h, d, dtype, seed=9, variant="cff")
    outs = K.fuse_chunks(cache, K.FusionConfig(threshold=0.8, variant="cff"), chunk, keep_samples=False)
    C, bpc = O.cff_chunks(p, t, chunk)
    _check_exact(outs, Kh, Vh, B * C, bpc, 0.8, O.cff_groups(B, C, None))


def test_exact_deep_tree_many_levels():
    """Deep trees (B = 32 rows, 5 levels) exercise shadow rows of absorbers that
    absorb again and are themselves absorbed later."""
    L, B, p, t, h, d = 1, 32, 16, 16, 1, 128
    cache, Kh, Vh = _cache(L, B, p, t, h, d, torch.bfloat16, seed=77)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.75), keep_samples=False)
    st = outs[0].fused.state
    assert int(st.shadow_count.item()) > 0
    _check_exact(outs, Kh, Vh, B, p, 0.75)


def test_exact_off_matches_stored_precision():
    """exact=False keeps the round-1 behaviour (re-scores read the stored bf16
    blocks); the tables may then differ from the reference near the threshold,
    but never outside the documented 1e-3 band."""
    from paper_2601_03067_b200.engine import FusionEngine
    from paper_2601_03067_b200.schedule import bff_plan

    L, B, p, t, h, d = 1, 8, 24, 16, 2, 128
    cache, Kh, Vh = _cache(L, B, p, t, h, d, torch.bfloat16, seed=31)
    eng = FusionEngine(cache.geometry(0), bff_plan(B, p, None), torch.bfloat16, "cuda", exact=False)
    pk, pv = cache.keys_dev.clone().reshape(-1), cache.values_dev.clone().reshape(-1)
    st = eng.run(pk, pv, 0.8)
    assert not st.exact and st.shadow_count is None
    ref = O.fuse_unit(O.layer_unit(Kh, 0), O.layer_unit(Vh, 0), B, p, 0.8,
                      gpu_absorber=st.absorber[0].cpu().numpy(), eps=1e-3, keep_samples=False)
    assert ref.mismatches == 0


def _seed_cache(cfg, seed):
    L, B, p, t, h, d = cfg
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.float32, seed=seed)
    return Kt, Vt


def test_cfg1_full_shape_vs_installed_reference():
    """BASELINE configs[0] at full shape, the same fp32 bytes on both sides:
    the device fuse_batch and the unmodified reference fuse_batch agree on every
    table entry, refcount, event and survivor, and on the compression ratio."""
    L, B, p, t, h, d = 4, 8, 64, 16, 8, 128
    Kt, Vt = _seed_cache((L, B, p, t, h, d), seed=1000)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), keep_samples=False)
    assert outs[0].fused.state.path_name == "tcgen05-split3"
    Kh, Vh = Kt.double().cpu().numpy(), Vt.double().cpu().numpy()
    ref = reference_fuse(Kh, Vh, dict(L=L, B=B, p=p, t=t, h=h, d=d), 0.8)
    before = after = rb = ra = 0
    for oc, ro in zip(outs, ref):
        tab = oc.fused.table
        assert oc.report.layer == ro.report.layer
        want = np.array([ro.fused.table.entries[(i, j)] for i in range(B) for j in range(p)])
        np.testing.assert_array_equal(tab.device_table.cpu().numpy(), want)
        assert dict(tab.refcount) == ro.fused.table.refcount
        assert oc.report.to_dict()["fused_events"] == ro.report.to_dict()["fused_events"]
        assert tuple(oc.fused.keys.phys_ids) == ro.fused.keys.phys_ids
        assert oc.report.merge_calls == ro.report.merge_calls
        assert oc.report.tree_depth == ro.report.tree_depth
        np.testing.assert_allclose(oc.fused.keys.directions, ro.fused.keys.directions, atol=2e-6)
        np.testing.assert_allclose(oc.fused.values.directions, ro.fused.values.directions, atol=2e-6)
        before += oc.report.blocks_before
        after += oc.report.blocks_after
        rb += ro.report.blocks_before
        ra += ro.report.blocks_after
    assert (before, after) == (rb, ra)
    assert before / after == pytest.approx(rb / ra, abs=0)


def test_cfg1_bf16_layer_vs_installed_reference():
    """The serving dtype at the cfg1 shape: a bf16 cache fused in exact mode
    equals the reference run on the same bf16 values widened to float64."""
    L, B, p, t, h, d = 2, 8, 64, 16, 8, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1000)
    cache = K.PagedKvCache(K.CacheDims(B=B, p=p, t=t, h=h, d=d, L=L), Kt, Vt)
    outs = K.fuse_batch(cache, K.FusionConfig(threshold=0.8), keep_samples=False)
    assert outs[0].fused.state.exact
    ref = reference_fuse(Kt.double().cpu().numpy(), Vt.double().cpu().numpy(),
                         dict(L=L, B=B, p=p, t=t, h=h, d=d), 0.8)
    for oc, ro in zip(outs, ref):
        want = np.array([ro.fused.table.entries[(i, j)] for i in range(B) for j in range(p)])
        np.testing.assert_array_equal(oc.fused.table.device_table.cpu().numpy(), want)
        assert oc.report.to_dict()["fused_events"] == ro.report.to_dict()["fused_events"]
        assert oc.report.blocks_after == ro.report.blocks_after


def test_path_names():
    L, B, p, t, h, d = 1, 4, 8, 16, 2, 64
    for dtype, name in ((torch.bfloat16, "tcgen05"), (torch.float32, "tcgen05-split3"),
                        (torch.float64, "simt")):
        cache, _, _ = _cache(L, B, p, t, h, d, dtype, seed=1)
        st = K.fuse_batch(cache, K.FusionConfig(threshold=0.8))[0].fused.state
        assert st.path_name == name
    # the CUDA-core path stays selectable for float32 (head dims that are not a multiple of 64)
    cache, _, _ = _cache(L, B, p, t, h, 32, torch.float32, seed=1)
    assert K.fuse_batch(cache, K.FusionConfig(threshold=0.8))[0].fused.state.path_name == "simt"
    assert N.PATH_TC == 2
