"""Generate golden vectors from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the reference kvfuse package read-only from
/root/reference/pkg/src, runs it on the reference's own fixtures and test
cases (pkg/tests/test_fusion.py, test_core.py, test_attention.py,
test_acceptance.py criteria 01/02/03/08) and writes their inputs and outputs
to tests/golden/golden.npz + golden.json. Those files are committed; nothing
at test time reads /root/reference.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    import kvfuse
    from kvfuse.attention import AttentionQuery, paged_attention
    from kvfuse.core import CacheDims, LayerView, PagedKvCache, UnfoldedLayer, refold, unfold_bff
    from kvfuse.fusion import (AdaptPolicy, FusionConfig, FusionReport, fast_fusion, fuse_batch,
                               fuse_chunks, reports_to_csv, tune_threshold)
    from kvfuse.workload import generate_fixture

    arrays: dict[str, np.ndarray] = {}
    cases: list[dict] = []

    def outcome_record(name: str, oc, dims_rows: int, bpr: int) -> dict:
        t = oc.table
        n = dims_rows * bpr
        table = np.array([t.entries[(s // bpr, s % bpr)] for s in range(n)], dtype=np.int64)
        ref = np.zeros(n, dtype=np.int64)
        for p_, c in t.refcount.items():
            ref[p_] = c
        arrays[f"{name}/table"] = table
        arrays[f"{name}/refcount"] = ref
        arrays[f"{name}/kdir"] = np.asarray(oc.fused.keys.directions)
        arrays[f"{name}/vdir"] = np.asarray(oc.fused.values.directions)
        arrays[f"{name}/samples"] = np.asarray(oc.report.similarity_samples)
        recs = []
        for m in oc.report.merge_records:
            mu, sd = m.moments()
            s = m.samples
            recs.append(dict(level=m.level, left=m.left_blocks, right=m.right_blocks,
                             fused=m.fused_count, n=int(s.size), mean=mu, std=sd,
                             min=float(s.min()) if s.size else 0.0,
                             max=float(s.max()) if s.size else 0.0))
        return dict(
            name=name,
            phys_ids=list(oc.fused.keys.phys_ids),
            report=oc.report.to_dict(),
            records=recs,
            reusable=sorted(int(x) for x in t.reusable),
            block_shape=list(oc.fused.block_shape),
        )

    # 1. acceptance 01: fast_fusion on every fixture layer x threshold
    acc01 = {
        "clusters1": (0.5, 0.9, 0.99),
        "orthogonal": (0.1, 0.5, 0.9),
        "clusters4": (0.88, 0.91, 0.93),
        "cff": (0.8, 0.9, 0.95),
    }
    for fx, thrs in acc01.items():
        cache = generate_fixture(fx)
        d = cache.dims
        arrays[f"fixture/{fx}/keys"] = cache.keys
        arrays[f"fixture/{fx}/values"] = cache.values
        for layer in range(d.L):
            keys, values = unfold_bff(cache, layer)
            for thr in thrs:
                oc = fast_fusion(keys, values, thr=thr)
                name = f"ff/{fx}/L{layer}/thr{thr}"
                rec = outcome_record(name, oc, d.B, d.p)
                rec.update(kind="fast_fusion_fixture", fixture=fx, layer=layer, thr=thr)
                cases.append(rec)

    # 2. test_fusion TestOracleReplay.test_random_rows_match
    for seed in range(4):
        rng = np.random.default_rng(seed)
        key_rows = rng.standard_normal((8, 3, 4))
        value_rows = rng.standard_normal((8, 3, 4))
        arrays[f"rows/{seed}/k"] = key_rows
        arrays[f"rows/{seed}/v"] = value_rows
        for thr in (0.1, 0.3, 0.6):
            def ul(rows):
                nrm = np.linalg.norm(rows, axis=-1)
                safe = np.where(nrm > 0, nrm, 1.0)
                return UnfoldedLayer(vectors=rows / safe[..., None], norms=nrm)
            oc = fast_fusion(ul(key_rows), ul(value_rows), thr=thr)
            name = f"rows/{seed}/thr{thr}"
            rec = outcome_record(name, oc, 8, 3)
            rec.update(kind="fast_fusion_rows", seed=seed, thr=thr)
            cases.append(rec)

    # 3. fuse_batch over fixtures (+ group_size) and tree structure
    for fx, thr, gs in (("clusters4", 0.91, None), ("clusters4", 0.9, 4), ("clusters1", 0.9, None)):
        cache = generate_fixture(fx)
        cfg = FusionConfig(threshold=thr, group_size=gs)
        for oc in fuse_batch(cache, cfg):
            name = f"fb/{fx}/thr{thr}/gs{gs}/L{oc.report.layer}"
            rec = outcome_record(name, oc, cache.dims.B, cache.dims.p)
            rec.update(kind="fuse_batch", fixture=fx, thr=thr, group_size=gs, layer=oc.report.layer)
            cases.append(rec)
    for B in (2, 3, 4, 5, 8, 13):
        dims = CacheDims(B=B, p=2, t=1, h=1, d=4, L=1)
        rng = np.random.default_rng(9)
        k = rng.standard_normal(dims.shape)
        v = rng.standard_normal(dims.shape)
        arrays[f"tree/{B}/keys"] = k
        arrays[f"tree/{B}/values"] = v
        oc = fuse_batch(PagedKvCache(dims=dims, keys=k, values=v), FusionConfig(threshold=0.5))[0]
        rec = outcome_record(f"tree/{B}", oc, B, 2)
        rec.update(kind="tree", B=B, thr=0.5)
        cases.append(rec)

    # 4. fuse_chunks on the cff fixture
    cache = generate_fixture("cff")
    for thr in (0.8, 0.9):
        for oc in fuse_chunks(cache, FusionConfig(threshold=thr, variant="cff"), 32):
            C = (cache.dims.p * cache.dims.t) // 32
            name = f"fc/cff/thr{thr}/L{oc.report.layer}"
            rec = outcome_record(name, oc, cache.dims.B * C, cache.dims.p // C)
            rec.update(kind="fuse_chunks", fixture="cff", thr=thr, chunk_tokens=32, layer=oc.report.layer)
            cases.append(rec)

    # 5. hand-derived merges (test_fusion.py:52-97)
    theta = math.radians(30.0)
    hand = {
        "bisector": ([[[1.0, 0.0]], [[math.cos(theta), math.sin(theta)]]], 0.8),
        "strict": ([[[1.0, 0.0]], [[math.cos(theta), math.sin(theta)]]], math.cos(theta)),
        "first_row_wins": ([[[1.0, 0.05]], [[2.0, 0.1]], [[0.5, 0.025]], [[3.0, 0.15]]], 0.99),
        "zero_blocks": ([[[0.0, 0.0], [1.0, 0.0]], [[0.0, 0.0], [1.0, 0.0]]], 0.5),
    }
    for hname, (rows, thr) in hand.items():
        arr = np.asarray(rows, dtype=np.float64)
        nrm = np.linalg.norm(arr, axis=-1)
        safe = np.where(nrm > 0, nrm, 1.0)
        layer = UnfoldedLayer(vectors=arr / safe[..., None], norms=nrm)
        arrays[f"hand/{hname}/rows"] = arr
        oc = fast_fusion(layer, layer, thr=thr)
        rec = outcome_record(f"hand/{hname}", oc, arr.shape[0], arr.shape[1])
        rec.update(kind="hand", hname=hname, thr=thr)
        cases.append(rec)

    # 6. refold + paged attention (test_core TestRefold, test_attention, acceptance 03)
    cache = generate_fixture("clusters4")
    oc = fuse_batch(cache, FusionConfig(threshold=0.91))[0]
    view = refold(oc.fused)
    arrays["refold/clusters4/thr0.91/L0/keys"] = view.keys
    arrays["refold/clusters4/thr0.91/L0/values"] = view.values
    rng = np.random.default_rng(17)
    att = []
    for i in range(6):
        q = rng.standard_normal(cache.dims.d)
        head = int(rng.integers(cache.dims.h))
        row = int(rng.integers(cache.dims.B))
        out_f, s_f = paged_attention(AttentionQuery(q=q, head=head), view, row)
        base = LayerView(keys=cache.keys[0], values=cache.values[0])
        out_b, s_b = paged_attention(AttentionQuery(q=q, head=head), base, row)
        arrays[f"att/{i}/q"] = q
        arrays[f"att/{i}/out_fused"] = out_f
        arrays[f"att/{i}/probs_fused"] = s_f.probs
        arrays[f"att/{i}/out_base"] = out_b
        arrays[f"att/{i}/probs_base"] = s_b.probs
        att.append(dict(i=i, head=head, row=row))

    # 7. threshold controller (acceptance 11) and report serialization (test_fusion.py:331-360)
    policy = AdaptPolicy(mode="target-compression", target=2.0, step=0.001,
                         min_threshold=0.85, max_threshold=0.97)
    thr, history = tune_threshold(generate_fixture("clusters4"), FusionConfig(threshold=0.90), policy,
                                  rel_tol=0.1, max_iters=30)
    reports = [o.report for o in fuse_batch(generate_fixture("clusters4"), FusionConfig(threshold=0.91))]
    agg = FusionReport.aggregate(reports)
    host = dict(tune=dict(final=thr, history=history), csv=reports_to_csv(reports),
                json=[r.to_json() for r in reports], aggregate=agg.to_dict())

    meta = dict(reference_version=kvfuse.__version__, numpy=np.__version__, cases=cases,
                attention=att, host=host)
    np.savez_compressed(OUT / "golden.npz", **arrays)
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(cases)} cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
