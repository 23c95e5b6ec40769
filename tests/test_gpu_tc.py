"""tcgen05 similarity path (bf16): cross-check against the CUDA-core path and
the float64 oracle at production block shapes (r = 16 * 8 * 128 folded,
partial tiles, per-head r = 2048)."""

import numpy as np
import pytest
import torch

import kvfuse_oracle as O

pytestmark = pytest.mark.gpu

K = pytest.importorskip("paper_2601_03067_b200")
from paper_2601_03067_b200 import _native as N  # noqa: E402
from paper_2601_03067_b200.engine import FusionEngine  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402


def _run(Kt, Vt, geom, plan, thr, path):
    eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device, path)
    return eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), thr, keep_samples=True)


@pytest.mark.parametrize("shape,head_mode", [
    ((2, 4, 48, 16, 8, 128), 0),   # folded r = 16384, 192 blocks/layer: partial M and N tiles
    ((1, 8, 64, 16, 8, 128), 1),   # per-head r = 2048
    ((1, 6, 100, 4, 2, 64), 0),    # odd sizes, r = 512
])
def test_tc_matches_simt_and_oracle(shape, head_mode):
    L, B, p, t, h, d = shape
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=21)
    geom = K.Geometry(L, B * p, t, h, d, head_mode)
    plan = bff_plan(B, p, None)
    st_tc = _run(Kt, Vt, geom, plan, 0.8, N.PATH_TC)
    st_sm = _run(Kt, Vt, geom, plan, 0.8, N.PATH_SIMT)
    # level 1 sees identical inputs on both paths: both must match the float64
    # similarity of the bf16 inputs (fp32 accumulation error only)
    Kh, Vh = Kt.double().cpu().numpy(), Vt.double().cpu().numpy()
    fa, fb = st_tc.level_samples[0].cpu().numpy(), st_sm.level_samples[0].cpu().numpy()
    assert np.array_equal(np.isnan(fa), np.isnan(fb))
    lv = plan.levels[0]
    off = 0
    errs = {"tc": 0.0, "simt": 0.0}
    for (lb, mid, re) in lv.merges.tolist():
        n = (mid - lb) * (re - mid)
        for u in range(geom.units):
            layer, head = (u // h, u % h) if head_mode else (u, None)
            X = O.layer_unit(Kh, layer, head)
            Xn = X / np.linalg.norm(X, axis=1, keepdims=True)
            exact = (Xn[lb:mid] @ Xn[mid:re].T).ravel()
            for name, f in (("tc", fa), ("simt", fb)):
                got = f[u, off:off + n]
                errs[name] = max(errs[name], float(np.abs(got - exact).max()))
        off += n
    # tensor-core fp32 accumulation: ~1e-4 relative worst case at r = 16K
    # (near-threshold pairs are re-scored exactly); CUDA-core path ~1e-6
    assert errs["tc"] < 2e-4 and errs["simt"] < 1e-5, errs
    for u in range(geom.units):
        layer, head = (u // h, u % h) if head_mode else (u, None)
        ref = O.fuse_unit(O.layer_unit(Kh, layer, head), O.layer_unit(Vh, layer, head), B, p, 0.8,
                          gpu_absorber=st_tc.absorber[u].cpu().numpy(), eps=1e-9, keep_samples=False)
        assert ref.mismatches == 0 and ref.flips == 0, ref.mismatch_detail  # exact mode
        np.testing.assert_array_equal(st_tc.table[u].cpu().numpy(), ref.table)
        np.testing.assert_array_equal(st_tc.refcount[u].cpu().numpy(), ref.refcount)


@pytest.mark.parametrize("shape,head_mode,compact_from,mode", [
    ((2, 16, 32, 16, 8, 128), 0, 1, "staged"),    # every level compacted
    ((2, 16, 32, 16, 8, 128), 0, 1, "gathered"),  # ... operands via TMA gather4
    ((1, 16, 40, 16, 8, 128), 0, 3, "staged"),    # top levels only, partial tiles
    ((1, 16, 40, 16, 8, 128), 0, 3, "gathered"),
    ((1, 13, 37, 16, 4, 64), 0, 1, "gathered"),   # odd sizes, d = 64
    ((1, 16, 24, 16, 2, 128), 1, 2, "staged"),    # per-head units
])
def test_tc_compaction_bitwise(shape, head_mode, compact_from, mode):
    """Compacted levels (alive rows staged densely, or gathered from the pool
    with TMA gather4) must reproduce the direct kernel's similarities bit for
    bit, hence identical decisions, tables and pools."""
    L, B, p, t, h, d = shape
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=9)
    geom = K.Geometry(L, B * p, t, h, d, head_mode)
    plan = bff_plan(B, p, None)
    outs = []
    for cf in (None, compact_from):
        # split-K sums partials in another order: compare compaction modes unsplit
        eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device, N.PATH_TC, compact_from=cf,
                           compact_mode=mode, split=False)
        assert eng.compact_from == cf
        outs.append(eng.run(Kt.clone().reshape(-1), Vt.clone().reshape(-1), 0.8, keep_samples=True))
    a, b = outs
    assert torch.equal(a.absorber, b.absorber)
    assert torch.equal(a.table, b.table)
    assert torch.equal(a.pool_k.view(torch.int16), b.pool_k.view(torch.int16))
    for sa, sb in zip(a.level_stats, b.level_stats):
        # counts / min / max exact; sums regroup across tiles -> fp rounding
        assert torch.equal(sa[..., [0, 1, 2, 3, 6, 7]], sb[..., [0, 1, 2, 3, 6, 7]])
        torch.testing.assert_close(sa[..., 4:6], sb[..., 4:6], rtol=1e-6, atol=1e-9)
    for xa, xb in zip(a.level_samples, b.level_samples):
        assert torch.equal(xa.isnan(), xb.isnan())
        assert torch.equal(torch.nan_to_num(xa), torch.nan_to_num(xb))
    assert a.live_count.sum() < L * B * p * (h if head_mode else 1)


@pytest.mark.parametrize("thr", [0.8, 0.9])
def test_tc_level1_exact_selection(thr):
    """Level 1 reads raw bf16 inputs and near-threshold pairs are re-scored in
    float64, so the device must take the float64 decision on every pair
    farther than 1e-9 from the threshold (no exemption band in practice)."""
    L, B, p, t, h, d = 1, 2, 256, 16, 8, 128
    Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=3)
    geom = K.Geometry(L, B * p, t, h, d, 0)
    plan = bff_plan(B, p, None)
    st = _run(Kt, Vt, geom, plan, thr, N.PATH_TC)
    Kh, Vh = Kt.double().cpu().numpy(), Vt.double().cpu().numpy()
    ref = O.fuse_unit(O.layer_unit(Kh, 0), O.layer_unit(Vh, 0), B, p, thr,
                      gpu_absorber=st.absorber[0].cpu().numpy(), eps=1e-9)
    assert ref.mismatches == 0 and ref.flips == 0
    got = st.level_samples[0][0].cpu().numpy()
    got = got[~np.isnan(got)]
    assert np.abs(got - ref.samples()).max() < 2e-4
