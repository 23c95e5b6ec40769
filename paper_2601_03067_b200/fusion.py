"""Batch / Chunks Fast-Fusion on the GPU -- the drop-in for kvfuse.fusion.

Same public names, arguments and errors as the reference (fusion.py:48-465):
FusionConfig, FusionEvent, MergeRecord, FusionReport, FusionOutcome,
fast_fusion, fuse_batch, fuse_chunks, adapt_threshold, tune_threshold.
The work runs in `engine.FusionEngine` (device kernels, level-synchronous
tree); reports are assembled lazily from device counters, so the host only
pays for what it reads.

Additions (keyword-only, defaults keep reference behaviour):
  FusionConfig.head_mode  "folded" (reference: one vector per block over all
                          heads) | "per_head" (one unit per layer x kv head)
  in_place=True           fuse the caller's device pool in place instead of a
                          private copy (the serving configuration)
  keep_samples            materialise MergeRecord.samples (O(pairs) memory);
                          default: only when the total is small
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .core import (
    BlockTable,
    FusedCache,
    FusedLayer,
    PagedKvCache,
    Slot,
    UnfoldedLayer,
    cff_layout,
    default_device,
)
from .engine import NONE, FusionEngine, FusionState, Geometry, acc_dtype, dtype_code
from .errors import ConfigError, CorruptionError, InsufficientDataError, InvalidCacheError
from .schedule import Plan, bff_plan, cff_plan, single_tree_plan

SAMPLES_AUTO_LIMIT = 1 << 22  # pairs across all units and levels


@dataclass(frozen=True)
class AdaptPolicy:
    """Threshold feedback rule (fusion.py:48-64)."""

    mode: str
    target: float
    step: float
    min_threshold: float
    max_threshold: float

    def __post_init__(self):
        if self.mode not in ("percentile", "target-compression"):
            raise ConfigError(f"unknown adapt mode {self.mode!r}")
        if self.step <= 0:
            raise ConfigError("adapt step must be positive")
        if not self.min_threshold < self.max_threshold:
            raise ConfigError("adapt bounds must satisfy min < max")


@dataclass(frozen=True)
class FusionConfig:
    """Threshold, variant and grouping of a fusion run (fusion.py:67-82)."""

    threshold: float
    variant: str = "bff"
    group_size: int | None = None
    adapt: AdaptPolicy | None = None
    head_mode: str = "folded"

    def __post_init__(self):
        if not -1.0 < self.threshold < 1.0:
            raise ConfigError(f"threshold must lie strictly inside (-1, 1), got {self.threshold}")
        if self.variant not in ("bff", "cff"):
            raise ConfigError(f"unknown fusion variant {self.variant!r}")
        if self.group_size is not None and self.group_size < 1:
            raise ConfigError("group_size must be >= 1")
        if self.head_mode not in ("folded", "per_head"):
            raise ConfigError(f"unknown head_mode {self.head_mode!r}")


@dataclass(frozen=True)
class FusionEvent:
    """One absorption: absorbing home slot and the home slots it consumed (fusion.py:85-90)."""

    absorber: Slot
    absorbed: tuple[Slot, ...]


class MergeRecord:
    """Similarity statistics of one tree merge (fusion.py:93-110).

    Carries the device moments (n, sum, sum of squares, min, max); ``samples``
    holds the raw similarities when they were materialised.
    """

    def __init__(self, level, left_blocks, right_blocks, samples, fused_count, *,
                 moments: tuple[float, float, float, float, float] | None = None):
        self.level = int(level)
        self.left_blocks = int(left_blocks)
        self.right_blocks = int(right_blocks)
        self.samples = np.asarray(samples, dtype=np.float64) if samples is not None else np.empty(0)
        self.fused_count = int(fused_count)
        if moments is None:
            s = self.samples
            moments = (
                float(s.size), float(s.sum()), float((s * s).sum()),
                float(s.min()) if s.size else 0.0, float(s.max()) if s.size else 0.0,
            )
        self._m = moments

    @property
    def n_samples(self) -> int:
        return int(self._m[0])

    @property
    def sample_sum(self) -> float:
        return self._m[1]

    @property
    def sample_sumsq(self) -> float:
        return self._m[2]

    @property
    def sample_min(self) -> float:
        return self._m[3]

    @property
    def sample_max(self) -> float:
        return self._m[4]

    def moments(self) -> tuple[float, float]:
        if self.samples.size:
            return float(np.mean(self.samples)), float(np.std(self.samples))
        n, s1, s2 = self._m[:3]
        if n == 0:
            return 0.0, 0.0
        mu = s1 / n
        return mu, math.sqrt(max(s2 / n - mu * mu, 0.0))

    def __repr__(self):
        return (f"MergeRecord(level={self.level}, left_blocks={self.left_blocks}, "
                f"right_blocks={self.right_blocks}, n={self.n_samples}, fused_count={self.fused_count})")


class FusionReport:
    """Per-unit outcome counters (fusion.py:113-171).

    ``fused_events``, ``similarity_samples`` and ``merge_records`` may be
    given directly (reference constructor) or produced lazily from the device
    state of a run.
    """

    def __init__(self, layer, blocks_before, blocks_after, fused_events, merge_calls, tree_depth,
                 similarity_samples, merge_records=None, *, head: int | None = None, _lazy=None):
        self.layer = layer
        self.blocks_before = int(blocks_before)
        self.blocks_after = int(blocks_after)
        self._events = fused_events
        self.merge_calls = int(merge_calls)
        self.tree_depth = int(tree_depth)
        self._samples = similarity_samples
        self._records = merge_records
        self.head = head
        self._lazy = _lazy  # object with .events(), .records(), .samples(), .summary()

    # lazily materialised fields ------------------------------------------
    @property
    def fused_events(self) -> list[FusionEvent]:
        if self._events is None:
            self._events = self._lazy.events()
        return self._events

    @fused_events.setter
    def fused_events(self, v):
        self._events = v

    @property
    def merge_records(self) -> list[MergeRecord]:
        if self._records is None:
            self._records = self._lazy.records() if self._lazy is not None else []
        return self._records

    @merge_records.setter
    def merge_records(self, v):
        self._records = v

    @property
    def similarity_samples(self) -> np.ndarray:
        if self._samples is None:
            self._samples = self._lazy.samples()
        return self._samples

    @similarity_samples.setter
    def similarity_samples(self, v):
        self._samples = v

    def device_samples(self) -> list | None:
        """Device sample rows (float64, NaN = masked pair) when the samples were
        kept on the GPU and not yet copied to the host, else None."""
        if self._samples is not None or self._lazy is None:
            return None
        fn = getattr(self._lazy, "device_samples", None)
        return fn() if fn is not None else None

    @property
    def samples_materialized(self) -> bool:
        return self._lazy is None or self._lazy.has_samples

    # reference API ---------------------------------------------------------
    @property
    def compression_ratio(self) -> float:
        return self.blocks_before / self.blocks_after

    @property
    def fused_blocks(self) -> int:
        if self._events is None and self._lazy is not None:
            return self.blocks_before - self.blocks_after
        return sum(len(e.absorbed) for e in self.fused_events)

    def similarity_summary(self) -> dict:
        """n / mean / population std / min / max of the merge similarities."""
        if self.samples_materialized:
            s = self.similarity_samples
            return {
                "n": int(s.size),
                "mean": float(np.mean(s)) if s.size else None,
                "std": float(np.std(s)) if s.size else None,
                "min": float(np.min(s)) if s.size else None,
                "max": float(np.max(s)) if s.size else None,
            }
        n = s1 = s2 = 0.0
        mn, mx = math.inf, -math.inf
        for m in self.merge_records:
            if m.n_samples:
                n += m.n_samples
                s1 += m.sample_sum
                s2 += m.sample_sumsq
                mn = min(mn, m.sample_min)
                mx = max(mx, m.sample_max)
        if n == 0:
            return {"n": 0, "mean": None, "std": None, "min": None, "max": None}
        mu = s1 / n
        return {"n": int(n), "mean": mu, "std": math.sqrt(max(s2 / n - mu * mu, 0.0)), "min": mn, "max": mx}

    def to_dict(self) -> dict:
        return {
            "layer": self.layer,
            "blocks_before": self.blocks_before,
            "blocks_after": self.blocks_after,
            "compression_ratio": self.compression_ratio,
            "merge_calls": self.merge_calls,
            "tree_depth": self.tree_depth,
            "fused_events": [
                [list(e.absorber), [list(s) for s in e.absorbed]] for e in self.fused_events
            ],
            "similarity": self.similarity_summary(),
        }

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True)

    @classmethod
    def aggregate(cls, reports: list["FusionReport"]) -> "FusionReport":
        """Collapse per-unit reports into one with layer -1 (fusion.py:158-171)."""
        parts = [r.device_samples() for r in reports]
        on_device = bool(reports) and all(p is not None for p in parts)
        all_mat = all(r.samples_materialized for r in reports)
        if on_device:  # keep them on the GPU; the host copy is built on first access
            samp = None
        elif all_mat:
            samples = [r.similarity_samples for r in reports if r.similarity_samples.size]
            samp = np.concatenate(samples) if samples else np.empty(0)
        else:
            samp = None
        out = cls(
            layer=-1,
            blocks_before=sum(r.blocks_before for r in reports),
            blocks_after=sum(r.blocks_after for r in reports),
            fused_events=None,  # concatenated on first access (_AggregateLazy)
            merge_calls=sum(r.merge_calls for r in reports),
            tree_depth=max((r.tree_depth for r in reports), default=0),
            similarity_samples=samp,
            merge_records=None if on_device else [m for r in reports for m in r.merge_records],
        )
        inner = None
        if on_device:
            inner = _DeviceParts([t for p in parts for t in p], reports)
        elif samp is None:
            inner = _NoSamples()
        out._lazy = _AggregateLazy(reports, inner)
        return out


class _AggregateLazy:
    """Aggregate report: the events of the parts are concatenated on first access (a
    threshold controller reading only the aggregate CR never builds the ~260K event
    objects of a cfg2 cache); samples / records come from `inner` when given."""

    def __init__(self, reports, inner):
        self.reports = reports
        self.inner = inner
        self.has_samples = inner.has_samples if inner is not None else True

    def events(self):
        return [e for r in self.reports for e in r.fused_events]

    def records(self):
        return self.inner.records() if self.inner is not None else []

    def samples(self):
        return self.inner.samples()

    def device_samples(self):
        fn = getattr(self.inner, "device_samples", None)
        return fn() if fn is not None else None


class _DeviceParts:
    """Aggregate of reports whose samples are still on the device."""

    has_samples = True

    def __init__(self, parts, reports):
        self.parts = parts
        self.reports = reports

    def device_samples(self):
        return self.parts

    def records(self):
        return [m for r in self.reports for m in r.merge_records]

    def samples(self):  # host copy in the reference's order (report, merge post-order)
        arrs = [r.similarity_samples for r in self.reports]
        arrs = [a for a in arrs if a.size]
        return np.concatenate(arrs) if arrs else np.empty(0)


class _NoSamples:
    has_samples = False

    def samples(self):
        raise InsufficientDataError(
            "similarity samples were not materialised (run with keep_samples=True)"
        )


CSV_HEADER = (
    "layer,blocks_before,blocks_after,compression_ratio,"
    "merge_calls,tree_depth,fused_blocks,sim_mean,sim_std"
)


def reports_to_csv(reports: list[FusionReport]) -> str:
    """One row per report (fusion.py:180-190)."""
    lines = [CSV_HEADER]
    for r in reports:
        s = r.similarity_summary()
        mu = s["mean"] if s["n"] else float("nan")
        sd = s["std"] if s["n"] else float("nan")
        lines.append(
            f"{r.layer},{r.blocks_before},{r.blocks_after},{r.compression_ratio:.6g},"
            f"{r.merge_calls},{r.tree_depth},{r.fused_blocks},{mu:.6g},{sd:.6g}"
        )
    return "\n".join(lines) + "\n"


@dataclass
class FusionOutcome:
    """Fused unit plus its report (fusion.py:193-202)."""

    fused: FusedCache
    report: FusionReport

    @property
    def table(self) -> BlockTable:
        return self.fused.table


# ---------------------------------------------------------------------------
# host views over a device FusionState
# ---------------------------------------------------------------------------
class _RunHost:
    """Host mirror of a FusionState, fetched once on first use."""

    def __init__(self, st: FusionState, keep_samples: bool):
        self.st = st
        self.keep_samples = keep_samples
        self._fetched = False

    def fetch(self):
        if self._fetched:
            return
        st = self.st
        self.live_count = st.live_count.cpu().numpy()
        self.stats = [s.cpu().numpy() for s in st.level_stats]
        self._absorber = None
        self._fetched = True

    def absorber(self) -> np.ndarray:
        if self._absorber is None:
            self._absorber = self.st.absorber.cpu().numpy()
        return self._absorber


class _UnitLazy:
    """Lazily rebuilds a unit's events / merge records / samples (reference order)."""

    def __init__(self, run: _RunHost, unit: int):
        self.run = run
        self.unit = unit
        self.has_samples = run.keep_samples

    def events(self) -> list[FusionEvent]:
        st = self.run.st
        plan: Plan = st.plan
        bpr = plan.bpr
        ab = self.run.absorber()[self.unit]
        js = np.nonzero(ab != NONE)[0]
        if js.size == 0:
            return []
        ls = ab[js].astype(np.int64)
        post = np.full(js.size, -1, dtype=np.int64)
        jrow = js // bpr
        for lv in plan.levels:
            m = lv.row_merge[jrow]
            ok = m >= 0
            mm = np.where(ok, m, 0)
            lb, mid, re = lv.merges[mm, 0], lv.merges[mm, 1], lv.merges[mm, 2]
            hit = ok & (ls >= lb) & (ls < mid) & (js >= mid) & (js < re) & (post < 0)
            post[hit] = lv.post[mm[hit]]
        order = np.lexsort((js, ls, post))
        events: list[FusionEvent] = []
        cur_key = None
        cur: list[Slot] = []
        for k in order:
            key = (int(post[k]), int(ls[k]))
            if key != cur_key:
                if cur_key is not None:
                    a = cur_key[1]
                    events.append(FusionEvent((a // bpr, a % bpr), tuple(cur)))
                cur_key, cur = key, []
            j = int(js[k])
            cur.append((j // bpr, j % bpr))
        a = cur_key[1]
        events.append(FusionEvent((a // bpr, a % bpr), tuple(cur)))
        return events

    def _merge_samples(self, li: int, m: int) -> np.ndarray:
        st = self.run.st
        smp = st.level_samples[li]
        if smp is None:
            return np.empty(0)
        lv = st.plan.levels[li]
        rect = lv.rect_sizes()
        off = int(rect[:m].sum())
        arr = smp[self.unit, off : off + int(rect[m])].cpu().numpy()
        return arr[~np.isnan(arr)]

    def records(self) -> list[MergeRecord]:
        self.run.fetch()
        plan: Plan = self.run.st.plan
        loc = {}
        for li, lv in enumerate(plan.levels):
            for m, post in enumerate(lv.post.tolist()):
                loc[post] = (li, m, lv.height)
        recs = []
        for post in range(plan.merge_calls):
            li, m, hgt = loc[post]
            s = self.run.stats[li][self.unit, m]
            samples = self._merge_samples(li, m) if self.has_samples else None
            recs.append(
                MergeRecord(hgt, s[0], s[1], samples, s[2], moments=(s[3], s[4], s[5], s[6], s[7]))
            )
        return recs

    def device_samples(self) -> list | None:
        if not self.has_samples:
            return None
        st = self.run.st
        return [smp[self.unit] for smp in st.level_samples if smp is not None]

    def samples(self) -> np.ndarray:
        if not self.has_samples:
            raise InsufficientDataError(
                "similarity samples were not materialised (run with keep_samples=True)"
            )
        arrs = [r.samples for r in self.records() if r.samples.size]
        return np.concatenate(arrs) if arrs else np.empty(0)


def _outcomes_from_state(st: FusionState, keep_samples: bool, rows: int, bpr: int,
                         block_shape: tuple[int, int, int], tables: list[BlockTable] | None = None,
                         layer_override: int | None = None, layer_offset: int = 0) -> list[FusionOutcome]:
    run = _RunHost(st, keep_samples)
    run.fetch()
    g = st.geom
    plan = st.plan
    outcomes = []
    acc_np = np.float64
    oknorm = st.orig_knorm.cpu().numpy().astype(acc_np)
    ovnorm = st.orig_vnorm.cpu().numpy().astype(acc_np)
    live_ids_all = st.live_ids
    for u in range(g.units):
        layer = ((u // g.h if g.head_mode else u) + layer_offset
                 if layer_override is None else layer_override)
        head = (u % g.h) if g.head_mode else None
        n_live = int(run.live_count[u])
        ids_dev = live_ids_all[u, :n_live]
        phys = ids_dev  # ascending live ids, materialised on access

        def loader(pool, norms, ids=ids_dev, u=u):
            out = torch.empty((ids.numel(), g.r), dtype=acc_dtype(pool.dtype), device=pool.device)
            N.call(
                "kvf_gather_vectors", N.ptr(pool), dtype_code(pool.dtype), *g.args(), u,
                N.ptr(ids), ids.numel(), N.ptr(norms), None, N.ptr(out), N.stream_ptr(),
            )
            return out

        if tables is not None:
            table = tables[u]
        else:
            table = BlockTable(layer, rows, bpr, st.table[u], st.refcount[u], st.alive[u])
        table._listeners.append(lambda u=u: _refresh_scales(st, u))
        fused = FusedCache(
            keys=FusedLayer(phys, loader=lambda f=loader: f(st.pool_k, st.knorm)),
            values=FusedLayer(phys, loader=lambda f=loader: f(st.pool_v, st.vnorm)),
            key_norms=oknorm[u].reshape(rows, bpr),
            value_norms=ovnorm[u].reshape(rows, bpr),
            table=table,
            block_shape=block_shape,
            state=st,
            unit=u,
            layer=layer,
            head=head,
        )
        report = FusionReport(
            layer=layer,
            blocks_before=g.NB,
            blocks_after=n_live,
            fused_events=None,
            merge_calls=plan.merge_calls,
            tree_depth=plan.tree_depth,
            similarity_samples=None,
            merge_records=None,
            head=head,
            _lazy=_UnitLazy(run, u),
        )
        outcomes.append(FusionOutcome(fused=fused, report=report))
    return outcomes


def _refresh_scales(st: FusionState, u: int) -> None:
    """Per-slot K / V scales of unit u from its current table (kvf_finalize without the
    live / free lists: the FusedCache keeps its post-fusion survivors, as the
    reference's frozen FusedLayer does after a later BlockTable.redirect)."""
    g = st.geom
    N.call(
        "kvf_finalize", dtype_code(st.pool_k.dtype), u, 1, g.NB, N.ptr(st.orig_knorm),
        N.ptr(st.orig_vnorm), N.ptr(st.knorm), N.ptr(st.vnorm), N.ptr(st.table), N.ptr(st.alive),
        N.ptr(st.k_scale), N.ptr(st.v_scale), None, None, None, None, N.stream_ptr(),
    )


def _want_samples(keep_samples, plan: Plan, units: int) -> bool:
    if keep_samples is not None:
        return bool(keep_samples)
    total = sum(int(lv.rect_sizes().sum()) for lv in plan.levels) * units
    return total <= SAMPLES_AUTO_LIMIT


def _pools(cache: PagedKvCache, in_place: bool, l0: int = 0, l1: int | None = None):
    k, v = cache.keys_dev[l0:l1], cache.values_dev[l0:l1]
    if in_place:
        return k, v
    return k.clone(), v.clone()


def _head_mode(cfg: FusionConfig) -> int:
    return 1 if cfg.head_mode == "per_head" else 0


STREAM_LAYERS = 4  # layers per H2D chunk when streaming a host-resident cache


def _stream_chunks(L: int) -> list[tuple[int, int]]:
    """Layer ranges streamed to the GPU: STREAM_LAYERS at a time, the last ones halved
    (..., 4, 2, 1, 1) so the fusion left after the final copy is one layer's."""
    out, c0 = [], 0
    while L - c0 > STREAM_LAYERS:
        out.append((c0, c0 + STREAM_LAYERS))
        c0 += STREAM_LAYERS
    n = L - c0
    while n > 1:
        h = (n + 1) // 2
        out.append((c0, c0 + h))
        c0, n = c0 + h, n - h
    if n == 1:
        out.append((c0, c0 + 1))
    return out


def _layer_range(layers, L: int) -> tuple[int, int]:
    """(first, stop) of a contiguous layer selection (a range, e.g. dist.shard_units)."""
    if layers is None:
        return 0, L
    ls = list(layers)
    if not ls:
        raise ConfigError("layers selects no layer")
    l0, l1 = ls[0], ls[-1] + 1
    if ls != list(range(l0, l1)) or l0 < 0 or l1 > L:
        raise ConfigError(f"layers must be a contiguous range inside [0, {L}), got {layers!r}")
    return l0, l1


def _run_fusion(cache: PagedKvCache, plan: Plan, hm: int, threshold: float, in_place: bool,
                keep_samples: bool, path: int, layers=None) -> list[tuple[FusionState, int]]:
    """Fuse the units of the selected layers (all by default); returns (state, first
    layer) per engine run.

    Device-resident caches run as one engine pass over the layer range (a view of
    the pool: layers are the outermost dimension). Host-resident caches
    (PagedKvCache(..., defer_upload=True)) stream to the GPU in chunks of
    STREAM_LAYERS layers on a copy stream while earlier chunks fuse on the
    current stream; every chunk is validated for NaN / Inf on the device.
    """
    l0, l1 = _layer_range(layers, cache.dims.L)
    if not cache.host_resident:
        d = cache.dims
        pk, pv = _pools(cache, in_place, l0, l1)
        geom = Geometry(l1 - l0, d.B * d.p, d.t, d.h, d.d, hm)
        engine = FusionEngine(geom, plan, pk.dtype, pk.device, path)
        return [(engine.run(pk.reshape(-1), pv.reshape(-1), threshold, keep_samples=keep_samples), l0)]
    d = cache.dims
    dev = cache.device
    shape = (l1 - l0,) + tuple(d.shape[1:])
    kd = torch.empty(shape, dtype=cache.dtype, device=dev)
    vd = torch.empty(shape, dtype=cache.dtype, device=dev)
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    copy.wait_stream(compute)  # kd / vd allocated on the compute stream
    chunks = _stream_chunks(l1 - l0)
    ready = []
    with torch.cuda.stream(copy):
        for c0, c1 in chunks:
            kd[c0:c1].copy_(cache.keys[l0 + c0:l0 + c1], non_blocking=True)
            vd[c0:c1].copy_(cache.values[l0 + c0:l0 + c1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
            ready.append(ev)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    engines: dict[int, FusionEngine] = {}
    out = []
    dt = dtype_code(cache.dtype)
    for (c0, c1), ev in zip(chunks, ready):
        compute.wait_event(ev)
        kc, vc = kd[c0:c1], vd[c0:c1]
        N.call("kvf_count_nonfinite", N.ptr(kc), dt, kc.numel(), N.ptr(bad), N.stream_ptr())
        N.call("kvf_count_nonfinite", N.ptr(vc), dt, vc.numel(), N.ptr(bad), N.stream_ptr())
        nl = c1 - c0
        if nl not in engines:
            engines[nl] = FusionEngine(Geometry(nl, d.B * d.p, d.t, d.h, d.d, hm), plan, cache.dtype,
                                       dev, path)
        st = engines[nl].run(kc.reshape(-1), vc.reshape(-1), threshold, keep_samples=keep_samples)
        out.append((st, l0 + c0))
    kd.record_stream(copy)
    vd.record_stream(copy)
    if int(bad.item()):
        raise InvalidCacheError("cache contains NaN or Inf entries")
    if in_place and (l0, l1) == (0, d.L):
        cache.keys_dev, cache.values_dev = kd, vd
    return out


def _audit_runs(runs) -> None:
    """Post-fusion table audit of every unit (the reference audits each layer after
    fusion, fusion.py:305 / 315, core.py:232-241): refcounts must equal the slot
    counts and only live blocks may be referenced. One device pass per run."""
    from .engine import audit

    for st, _ in runs:
        g = st.geom
        if not audit(st.table, st.refcount, st.alive, g.units, g.NB):
            raise CorruptionError("refcounts inconsistent with logical slot mapping")


def _outcomes(runs, keep_samples, rows, bpr, shape, check: bool = True) -> list[FusionOutcome]:
    if check:
        _audit_runs(runs)
    outs: list[FusionOutcome] = []
    for st, c0 in runs:
        outs.extend(_outcomes_from_state(st, keep_samples, rows, bpr, shape, layer_offset=c0))
    return outs


def fuse_batch(cache: PagedKvCache, cfg: FusionConfig, *, in_place: bool = False,
               keep_samples: bool | None = None, path: int = N.PATH_AUTO,
               audit: bool = True, layers=None) -> list[FusionOutcome]:
    """Batch Fast-Fusion across requests, all layers at once (fusion.py:360-374).

    Returns one outcome per layer (folded) or per (layer, kv head) in
    per-head mode, layer-major. ``audit`` runs the device table audit after
    fusion and raises CorruptionError on an inconsistent table, as the
    reference does per layer (fusion.py:315). ``layers`` (a contiguous range,
    e.g. ``dist.shard_units(L, world, rank)``) fuses only those layers -- layers
    are independent (fusion.py:367-374), so a shard's outcomes equal the
    full run's for the same layers; report.layer keeps the cache index.
    """
    if cfg.variant != "bff":
        raise ConfigError(f"fuse_batch requires variant 'bff', got {cfg.variant!r}")
    dims = cache.dims
    hm = _head_mode(cfg)
    geom = cache.geometry(hm)
    plan = bff_plan(dims.B, dims.p, cfg.group_size)
    ks = _want_samples(keep_samples, plan, geom.units)
    runs = _run_fusion(cache, plan, hm, cfg.threshold, in_place, ks, path, layers)
    shape = (dims.t, 1, dims.d) if hm else (dims.t, dims.h, dims.d)
    return _outcomes(runs, ks, dims.B, dims.p, shape, check=audit)


def fuse_chunks(cache: PagedKvCache, cfg: FusionConfig, chunk_tokens: int, *,
                in_place: bool = False, keep_samples: bool | None = None,
                path: int = N.PATH_AUTO, audit: bool = True, layers=None) -> list[FusionOutcome]:
    """Chunks Fast-Fusion across the chunks of each request (fusion.py:377-415).

    Rows are (request, chunk); trees never cross requests; physical blocks
    shared after fusion are flagged reusable.
    """
    if cfg.variant != "cff":
        raise ConfigError(f"fuse_chunks requires variant 'cff', got {cfg.variant!r}")
    dims = cache.dims
    C, bpc = cff_layout(dims.p, dims.t, chunk_tokens)
    hm = _head_mode(cfg)
    geom = cache.geometry(hm)
    plan = cff_plan(dims.B, C, bpc, cfg.group_size)
    ks = _want_samples(keep_samples, plan, geom.units)
    runs = _run_fusion(cache, plan, hm, cfg.threshold, in_place, ks, path, layers)
    shape = (dims.t, 1, dims.d) if hm else (dims.t, dims.h, dims.d)
    outcomes = _outcomes(runs, ks, dims.B * C, bpc, shape, check=audit)
    for oc in outcomes:  # reusable = {refcount > 1} (fusion.py:409-411)
        ref = oc.fused.table.device_refcount.cpu().numpy()
        oc.fused.table.reusable = set(int(p) for p in np.nonzero(ref > 1)[0])
    return outcomes


def fast_fusion(keys: UnfoldedLayer, values: UnfoldedLayer, thr: float,
                table: BlockTable | None = None, layer: int = 0,
                block_shape: tuple[int, int, int] | None = None, *,
                keep_samples: bool | None = None, path: int = N.PATH_AUTO) -> FusionOutcome:
    """One tree over all rows of one unfolded layer (fusion.py:339-351)."""
    if not -1.0 < thr < 1.0:
        raise ConfigError(f"threshold must lie strictly inside (-1, 1), got {thr}")
    kv, vv = keys.vectors, values.vectors
    if tuple(vv.shape) != tuple(kv.shape):
        raise ConfigError("keys and values must be row-aligned")
    rows, bpr, r = keys.rows, keys.blocks_per_row, keys.r
    dev = default_device()

    def dev_tensor(x, dtype=None):
        if isinstance(x, torch.Tensor):
            return x.to(dev)
        return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(dev)

    kvec, vvec = dev_tensor(kv), dev_tensor(vv)
    kn, vn = dev_tensor(keys.norms), dev_tensor(values.norms)
    if kvec.dtype not in (torch.float64, torch.float32, torch.bfloat16):
        kvec, vvec = kvec.double(), vvec.double()
    acc = acc_dtype(kvec.dtype)
    # the pool holds raw blocks: direction * norm (reference keeps them split)
    pk = (kvec.to(acc) * kn.to(acc)[..., None]).to(kvec.dtype).contiguous().reshape(-1)
    pv = (vvec.to(acc) * vn.to(acc)[..., None]).to(vvec.dtype).contiguous().reshape(-1)
    # the pool holds each row as a (t, h, d) block when the caller names one (attention
    # over the fused unit reads heads), else as one r-vector
    bt, bh, bd = block_shape if block_shape and int(np.prod(block_shape)) == r else (1, 1, r)
    geom = Geometry(1, rows * bpr, int(bt), int(bh), int(bd), 0)
    plan = single_tree_plan(rows, bpr)
    engine = FusionEngine(geom, plan, pk.dtype, dev, path)
    ks = _want_samples(keep_samples, plan, 1)
    tables = None
    kw = {}
    if table is not None:
        table.audit()
        n = rows * bpr
        if (table.rows * table.blocks_per_row != n
                or not torch.equal(table.device_table.cpu(), torch.arange(n, dtype=torch.int32))
                or not bool((table.device_refcount == 1).all())):
            raise ConfigError("fast_fusion requires an identity (pre-fusion) block table")
        kw = dict(table=table.device_table.view(1, n), refcount=table.device_refcount.view(1, n),
                  alive=table.device_alive.view(1, n))
        tables = [table]
    st = engine.run(pk, pv, thr, orig_knorm=kn.reshape(1, -1), orig_vnorm=vn.reshape(1, -1),
                    keep_samples=ks, **kw)
    if table is not None:
        table._dirty()
    _audit_runs([(st, 0)])  # fusion.py:305 (table.audit after the tree)
    shape = block_shape or (1, 1, r)
    return _outcomes_from_state(st, ks, rows, bpr, shape, tables=tables, layer_override=layer)[0]


def device_quantile(parts: list[torch.Tensor], q: float) -> float:
    """np.quantile(concat(non-NaN entries of parts), q) computed on the GPU
    (kvf_quantile: exact radix select, numpy's 'linear' interpolation)."""
    import ctypes as C

    parts = [t for t in parts if t is not None and t.numel()]
    if parts and any(t.dtype != torch.float64 or not t.is_cuda for t in parts):
        raise ConfigError("device_quantile takes float64 CUDA tensors")
    dev = parts[0].device if parts else torch.device("cuda")
    parts = [t.contiguous() for t in parts]
    ptrs = (C.c_void_p * max(len(parts), 1))(*[t.data_ptr() for t in parts])
    lens = (C.c_int64 * max(len(parts), 1))(*[t.numel() for t in parts])
    ws = torch.empty(int(N.lib().kvf_quantile_ws_bytes()), dtype=torch.uint8, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    N.call("kvf_quantile", ptrs, lens, len(parts), float(q), N.ptr(out), N.ptr(ws), ws.numel(),
           N.stream_ptr())
    v = float(out.item())
    if math.isnan(v):
        raise InsufficientDataError("percentile adaptation needs a nonempty similarity sample set")
    return v


def adapt_threshold(policy: AdaptPolicy, report: FusionReport, current: float) -> float:
    """One step of the threshold controller (fusion.py:418-437)."""
    if policy.mode == "target-compression":
        cr = report.compression_ratio
        if cr > policy.target:
            return min(current + policy.step, policy.max_threshold)
        if cr < policy.target:
            return max(current - policy.step, policy.min_threshold)
        return current
    dev = report.device_samples()
    if dev is not None:  # samples still on the GPU: exact quantile without a host copy
        q = device_quantile(dev, 1.0 - policy.target)
    else:
        samples = report.similarity_samples
        if samples.size == 0:
            raise InsufficientDataError("percentile adaptation needs a nonempty similarity sample set")
        q = float(np.quantile(samples, 1.0 - policy.target))
    return min(max(q, policy.min_threshold), policy.max_threshold)


def tune_threshold(cache: PagedKvCache, cfg: FusionConfig, policy: AdaptPolicy,
                   rel_tol: float = 0.1, max_iters: int = 30) -> tuple[float, list[tuple[float, float]]]:
    """Fuse + adapt until the aggregate CR is within rel_tol of target (fusion.py:440-465)."""
    if policy.mode != "target-compression":
        raise ConfigError("tune_threshold requires a target-compression policy")
    thr = cfg.threshold
    history: list[tuple[float, float]] = []
    for _ in range(max_iters):
        run_cfg = FusionConfig(threshold=thr, variant=cfg.variant, group_size=cfg.group_size,
                               head_mode=cfg.head_mode)
        outcomes = fuse_batch(cache, run_cfg, keep_samples=False)
        combined = FusionReport.aggregate([o.report for o in outcomes])
        cr = combined.compression_ratio
        history.append((thr, cr))
        if abs(cr - policy.target) / policy.target <= rel_tol:
            return thr, history
        thr = adapt_threshold(policy, combined, thr)
    return thr, history
