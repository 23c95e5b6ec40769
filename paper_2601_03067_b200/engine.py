"""Device fusion engine: runs the merge tree level by level on the GPU.

One `FusionState` holds the fusion state of U independent units that share a
merge plan (all layers -- and, in per-head mode, all KV heads -- of a cache).
Per tree level the engine issues four stream-ordered launches:

  kvf_similarity_select  K2+K3  similarity GEMM + first-match epilogue
  kvf_level_stats               MergeRecord counters + absorber marking
  kvf_merge_groups       K4     normalised-sum merge, written in place
  kvf_remap              K5     block table / refcount / alive update

and `kvf_finalize` afterwards derives per-slot K/V scales and the ascending
live / free block lists. Reference: _Engine (fusion.py:205-282) and
_fuse_layer (fusion.py:290-336), restated level-synchronously.
"""

from __future__ import annotations

import contextlib
import os

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError
from .schedule import Plan

NONE = 0x7FFFFFFF
# tcgen05 path: pairs with |sim - thr| <= band are re-decided in float64.
# RESCORE_BAND covers the fp32 accumulation of exact bf16 products (level 1 of a
# bf16 pool: original blocks; float32 pools through the hi/lo split, ~1e-6);
# RESCORE_BAND_WIDE also covers the bf16 rounding of fused blocks stored in the pool
# at levels >= 2 in exact mode, |sim_pool - sim_exact| <= ~3e-4 at r = 2048.
RESCORE_BAND = 2.0**-11
RESCORE_BAND_WIDE = 2.0**-8
RESCORE_CAP = 1 << 20

_DT = {torch.float64: N.DT_F64, torch.float32: N.DT_F32, torch.bfloat16: N.DT_BF16}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DT[dt]
    except KeyError:
        raise ConfigError(f"unsupported pool dtype {dt}; use float64, float32 or bfloat16") from None


def acc_dtype(dt: torch.dtype) -> torch.dtype:
    return torch.float64 if dt == torch.float64 else torch.float32


@dataclass(frozen=True)
class Geometry:
    """Pool (L, NB, t, h, d) and unit layout."""

    L: int
    NB: int
    t: int
    h: int
    d: int
    head_mode: int = 0  # 0 folded (unit = layer), 1 per_head (unit = layer*h + head)

    @property
    def units(self) -> int:
        return self.L * self.h if self.head_mode else self.L

    @property
    def r(self) -> int:
        return self.t * self.d if self.head_mode else self.t * self.h * self.d

    @property
    def E(self) -> int:
        return self.t * self.h * self.d

    def args(self):
        return (self.L, self.NB, self.t, self.h, self.d, self.head_mode)


def block_norms(pool: torch.Tensor, geom: Geometry, stream=None) -> torch.Tensor:
    """K1: per-(unit, block) L2 norms, Acc[U, NB] (core.py:115-119)."""
    out = torch.empty((geom.units, geom.NB), dtype=acc_dtype(pool.dtype), device=pool.device)
    N.call(
        "kvf_block_norms", N.ptr(pool), dtype_code(pool.dtype), *geom.args(), N.ptr(out),
        N.stream_ptr(stream),
    )
    return out


class _PlanDevice:
    """Device copies of one plan's per-level arrays (uploaded once)."""

    def __init__(self, plan: Plan, tm: int, tn: int, ppt: int, device):
        self.levels = []
        for lv in plan.levels:
            tiles, tile_off = lv.tiling(tm, tn)
            rect = lv.rect_sizes()
            s_off = np.concatenate([[0], np.cumsum(rect)[:-1]]).astype(np.int64)
            self.levels.append(
                dict(
                    merges=torch.from_numpy(lv.merges.copy()).to(device),
                    row_merge=torch.from_numpy(lv.row_merge.copy()).to(device),
                    tiles=torch.from_numpy(tiles.copy()).to(device),
                    tile_off=torch.from_numpy(tile_off.copy()).to(device),
                    # offsets in partials slots (ppt slots per tile)
                    tile_off_p=torch.from_numpy((tile_off * ppt).astype(np.int32)).to(device),
                    sample_off=torch.from_numpy(s_off).to(device),
                    nm=int(lv.merges.shape[0]),
                    nt=int(tiles.shape[0]),
                    rect_total=int(rect.sum()),
                )
            )


def _paired_level(base: dict, ppt: int, device) -> dict:
    """Device arrays of a level run as paired small merges (KVF_SIM_PAIRED): tile k =
    merges 2k and 2k + 1 on the diagonal of one pair tile; merge m owns partial slots
    [(m // 2) * ppt + (m % 2) * ppt / 2, + ppt / 2)."""
    nm = base["nm"]
    nt = (nm + 1) // 2
    tiles = np.zeros((nt, 3), dtype=np.int32)
    tiles[:, 0] = np.arange(0, nm, 2, dtype=np.int32)
    m = np.arange(nm + 1)
    off_p = ((m // 2) * ppt + (m % 2) * (ppt // 2)).astype(np.int32)
    d = dict(base)
    d.update(tiles=torch.from_numpy(tiles).to(device), tile_off=None,
             tile_off_p=torch.from_numpy(off_p).to(device), nt=nt, paired=True)
    return d


def _plan_device(plan: Plan, tm: int, tn: int, ppt: int, device) -> _PlanDevice:
    cache = plan.__dict__.setdefault("_device_cache", {})
    key = (tm, tn, ppt, str(device))
    if key not in cache:
        cache[key] = _PlanDevice(plan, tm, tn, ppt, device)
    return cache[key]


def tile_shape(dtype: torch.dtype, head_mode: int, path: int) -> tuple[int, int, int]:
    """(tile_m, tile_n, partials slots per tile) of a similarity path."""
    import ctypes as C

    tm, tn, ppt = C.c_int(), C.c_int(), C.c_int()
    N.call("kvf_sim_tile_shape", dtype_code(dtype), head_mode, path, C.byref(tm), C.byref(tn),
           C.byref(ppt))
    return tm.value, tn.value, ppt.value


@dataclass
class FusionState:
    """Device-resident result of fusing U units (all tensors [U, NB] unless noted)."""

    geom: Geometry
    plan: Plan
    threshold: float
    pool_k: torch.Tensor
    pool_v: torch.Tensor
    knorm: torch.Tensor  # stored norms of the (possibly rewritten) pool blocks
    vnorm: torch.Tensor
    orig_knorm: torch.Tensor  # per-slot original norms (FusedCache.key_norms)
    orig_vnorm: torch.Tensor
    fusable: torch.Tensor
    alive: torch.Tensor
    absorber: torch.Tensor  # event record: absorber[j] = l (or NONE)
    table: torch.Tensor  # slot -> physical block
    refcount: torch.Tensor
    k_scale: torch.Tensor | None = None
    v_scale: torch.Tensor | None = None
    live_ids: torch.Tensor | None = None
    live_count: torch.Tensor | None = None  # [U]
    free_ids: torch.Tensor | None = None
    free_count: torch.Tensor | None = None
    level_stats: list[torch.Tensor] = field(default_factory=list)  # per level [U, nm, 8]
    level_samples: list[torch.Tensor | None] = field(default_factory=list)
    launches: int = 0
    sim_events: list = field(default_factory=list)  # (start, end, level) CUDA events
    near_threshold: list = field(default_factory=list)  # per level int32[1]: re-scored pairs
    rescore_cap: int = 0
    path_name: str = ""  # "tcgen05" | "tcgen05-split3" (float32 hi/lo operands) | "simt"
    exact: bool = False  # decisions re-scored against float64-derived key directions
    shadow_count: torch.Tensor | None = None  # int32[1]: shadow slots taken (exact mode)
    shadow_cap: int = 0

    def inexact_pairs(self) -> int:
        """Near-threshold pairs that could not be re-scored (queue overflow) and were
        decided from the tensor-core value; 0 unless a level overflowed RESCORE_CAP."""
        if not self.rescore_cap:
            return 0
        return sum(max(0, int(c.item()) - self.rescore_cap) for c in self.near_threshold)

    def inexact_blocks(self) -> int:
        """Key absorbers without a shadow row (arena overflow; exact mode only)."""
        if self.shadow_count is None:
            return 0
        return max(0, int(self.shadow_count.item()) - self.shadow_cap)


@dataclass
class TilePlan:
    """Per-level similarity launch choices of a FusionEngine (host-only, no device state)."""

    compact_from: int | None
    paired: list  # two small merges per tile on the pair tile's diagonal (KVF_SIM_PAIRED)
    nsplit: list  # split-K factor
    wide: list  # 512 x 256 tile per CTA pair (KVF_PATH_TC_WIDE)
    nt: list  # tiles per unit of the chosen tiling
    fuse_knorm: bool  # level-1 launch writes the key norms (KVF_SIM_WRITE_NORMS)


def auto_compact_from(plan: Plan) -> int | None:
    """Lowest compacted tree height: depth - 1 (dead blocks are ~55% of the top merges'
    rectangles); one lower when those merges span >= COMPACT_BIG_MERGE blocks (their
    rectangle cost grows with the merge size while staging grows with the block count:
    cfg5 shape, heights 6-8 compacted 571 -> 534-547 ms per layer; heights 5-8: 551 ms)."""
    compact_from = plan.tree_depth - 1 if plan.tree_depth >= 4 else None
    if compact_from is not None and compact_from - 1 >= 2:
        lo = [lv for lv in plan.levels if lv.height == compact_from - 1]
        if lo and len(lo[0].merges) and int((lo[0].merges[:, 2] - lo[0].merges[:, 0]).min()) >= COMPACT_BIG_MERGE:
            compact_from -= 1
    return compact_from


def tile_plan(plan: Plan, geom: Geometry, dtype: torch.dtype, path: int, compact_from, compact_mode: str,
              split: bool, pairs: int, env=None) -> TilePlan:
    """Choose, per tree level, the similarity launch: paired small merges, split-K, the wide
    tile, and whether level 1 computes the key norms. Pure host logic over the plan
    (`env` defaults to os.environ: the KVF_SIM_* A/B knobs)."""
    env = os.environ if env is None else env
    U = geom.units
    filter_mode = path == N.PATH_TC and dtype == torch.float32
    if compact_from == "auto":
        compact_from = auto_compact_from(plan)
    if path != N.PATH_TC or geom.d % 8 != 0 or filter_mode:
        compact_from = None
    nlv = len(plan.levels)
    tp = TilePlan(compact_from, [False] * nlv, [1] * nlv, [False] * nlv, [0] * nlv, False)
    if path != N.PATH_TC:
        tm = tn = _simt_tile()
        for li, lv in enumerate(plan.levels):
            tp.nt[li] = int(lv.tiling(tm, tn)[0].shape[0])
        return tp
    tm, tn, _ = tile_shape(dtype, geom.head_mode, path)
    compacted = [compact_from is not None and lv.height >= compact_from for lv in plan.levels]
    for li, lv in enumerate(plan.levels):
        tp.nt[li] = int(lv.tiling(tm, tn)[0].shape[0])
        m_ = lv.merges
        # paired small merges: every merge side fits one 128-row box
        if (env.get("KVF_SIM_PAIRED", "1") != "0" and len(m_) >= 2 and not compacted[li]
                and int((m_[:, 1] - m_[:, 0]).max()) <= tm // 2 and int((m_[:, 2] - m_[:, 1]).max()) <= tn // 2):
            tp.paired[li] = True
            tp.nt[li] = (len(m_) + 1) // 2
    # split-K: few, long-K tiles (cfg1, CFF) spread over all SMs
    if split:
        nk = geom.r // 64 * (3 if filter_mode else 1)
        for li in range(nlv):
            if compacted[li] and compact_mode == "gathered":
                continue
            n_tiles = tp.nt[li] * U
            s_ = choose_split(n_tiles, nk, pairs)
            while s_ > 1 and n_tiles * s_ * _TILE_PART_BYTES > SPLIT_PART_BUDGET:
                s_ -= 1
            tp.nsplit[li] = s_
    # wide tiles where a level's merges fill 512 rows and it has two waves of them
    if geom.head_mode == 0 and compact_mode != "gathered":
        wide_env = env.get("KVF_SIM_WIDE", "auto")
        tmw, _, _ = tile_shape(dtype, 0, N.PATH_TC_WIDE)
        for li, lv in enumerate(plan.levels):
            if tp.nsplit[li] != 1 or wide_env == "0" or not len(lv.merges) or tp.paired[li]:
                continue
            left_min = int((lv.merges[:, 1] - lv.merges[:, 0]).min())
            nt_w = int(lv.tiling(tmw, tn)[0].shape[0])
            if wide_env == "1" or (left_min >= tmw and nt_w * U >= 2 * pairs):
                tp.wide[li] = True
                tp.nt[li] = nt_w
    # fused level-1 key norms: every block is an operand row of exactly one level-1 tile
    if dtype == torch.bfloat16 and nlv and env.get("KVF_FUSE_KNORM", "1") != "0":
        lv0 = plan.levels[0]
        m0 = lv0.merges
        tp.fuse_knorm = bool(
            len(m0) and tp.nsplit[0] == 1 and not tp.wide[0] and not compacted[0]
            and (lv0.row_merge >= 0).all()
            and int((m0[:, 1] - m0[:, 0]).max()) <= tm and int((m0[:, 2] - m0[:, 1]).max()) <= tn)
    return tp


def _simt_tile() -> int:
    return tile_shape(torch.float64, 0, N.PATH_SIMT)[0]


class FusionEngine:
    """Runs fusion of all units of a geometry for one plan (see module doc)."""

    def __init__(self, geom: Geometry, plan: Plan, dtype: torch.dtype, device, path: int = N.PATH_AUTO,
                 compact_from: int | None | str = "auto", compact_mode: str = "auto",
                 exact: bool | None = None, split: bool = True):
        if plan.n_blocks != geom.NB:
            raise ConfigError(f"plan covers {plan.n_blocks} blocks, geometry has {geom.NB}")
        self.geom = geom
        self.plan = plan
        self.dtype = dtype
        self.device = torch.device(device)
        if path == N.PATH_AUTO:
            tc = dtype in (torch.bfloat16, torch.float32) and tc_available(geom)
            path = N.PATH_TC if tc else N.PATH_SIMT
        if path == N.PATH_TC and dtype == torch.float64:
            raise ConfigError("the tcgen05 similarity path takes bf16 or float32 pools")
        self.path = path
        # float32 pools on the tensor cores: bf16 operand copy + float64 re-score
        self.filter_mode = path == N.PATH_TC and dtype == torch.float32
        # exact mode (bf16 pools): fp32 shadow rows of the fused key directions, so
        # re-scored decisions at levels >= 2 follow the reference's float64 directions
        if exact is None:  # exact mode covers r <= 16384; longer vectors merge on merge_long_kernel
            exact = path == N.PATH_TC and dtype == torch.bfloat16 and geom.r <= 16384 and geom.d % 8 == 0
        if exact and not (path == N.PATH_TC and dtype == torch.bfloat16):
            exact = False  # float32 / float64 pools keep fused keys at full precision already
        if exact and (geom.r > 16384 or geom.d % 8 != 0):
            raise ConfigError("exact mode needs r <= 16384 and d % 8 == 0 (use head_mode='per_head')")
        self.exact = bool(exact)
        self.tm, self.tn, self.ppt = tile_shape(dtype, geom.head_mode, path)
        self.pdev = _plan_device(plan, self.tm, self.tn, self.ppt, self.device)
        U, NB = geom.units, geom.NB
        dev = self.device
        # member counts / segments / absorber list of the current level
        self.level_ws = torch.zeros(int(N.lib().kvf_level_ws_ints(U * NB)), dtype=torch.int32,
                                    device=dev)
        pairs = 74
        if path == N.PATH_TC:
            pairs = max(1, torch.cuda.get_device_properties(self.device).multi_processor_count // 2)
        # compaction of the top levels (tcgen05 path: dead blocks dominate the upper merges'
        # rectangles, so their alive K rows are staged densely), paired / split-K / wide
        # launches per level and the fused level-1 norms: tile_plan (host logic)
        tp = tile_plan(plan, geom, dtype, path, compact_from, compact_mode, split, pairs)
        compact_from = tp.compact_from
        self.compact_from = compact_from
        self.paired, self.nsplit, self.wide, self.fuse_knorm = tp.paired, tp.nsplit, tp.wide, tp.fuse_knorm
        # exact float64 re-score of pairs within RESCORE_BAND of the threshold
        # (tensor-core fp32 accumulation error is ~1e-4 relative at r = 16K)
        self.rescore_cap = RESCORE_CAP if path == N.PATH_TC else 0
        self.rescore = (torch.empty(4 * (self.rescore_cap + 1), dtype=torch.int32, device=dev)
                        if self.rescore_cap else None)
        # hi / lo bf16 split of a float32 pool (kvf_convert_rows), 2 x the pool's elements
        self.filter = (torch.empty(2 * geom.L * NB * geom.E, dtype=torch.bfloat16, device=dev)
                       if self.filter_mode else None)
        # device tile lists of the chosen launches
        self.levels = list(self.pdev.levels)
        pdw = None
        for li in range(len(self.levels)):
            if self.paired[li]:
                self.levels[li] = _paired_level(self.levels[li], self.ppt, self.device)
            elif self.wide[li]:
                if pdw is None:
                    tmw, _, _ = tile_shape(dtype, 0, N.PATH_TC_WIDE)
                    pdw = _plan_device(plan, tmw, self.tn, self.ppt, self.device)
                self.levels[li] = pdw.levels[li]
        # split-K partials (fp32 accumulator tiles) and arrival counters
        self.split_part = self.split_count = None
        need = max([self.levels[li]["nt"] * U * s_ * _TILE_PART_BYTES
                    for li, s_ in enumerate(self.nsplit) if s_ > 1], default=0)
        if need:
            tiles_max = max(self.levels[li]["nt"] * U for li, s_ in enumerate(self.nsplit) if s_ > 1)
            self.split_part = torch.empty(need // 4, dtype=torch.float32, device=dev)
            self.split_count = torch.zeros(2 * tiles_max, dtype=torch.int32, device=dev)
        max_nt = max([lv["nt"] for lv in self.levels], default=1)
        self.partials = torch.empty((U, max(max_nt * self.ppt, 1), 5), dtype=torch.float64, device=dev)
        self.shadow = self.sidx = self.scount = None
        self.shadow_cap = 0
        if self.exact:
            # distinct key absorbers: U * NB / 2 bounds them unless absorbers are themselves
            # absorbed later; overflow is counted (FusionState.inexact_blocks), never silent
            self.shadow_cap = max(1, (U * NB + 1) // 2)
            self.shadow = torch.empty((self.shadow_cap, geom.r), dtype=torch.float32, device=dev)
            self.sidx = torch.empty((U, NB), dtype=torch.int32, device=dev)
            self.scount = torch.empty(1, dtype=torch.int32, device=dev)
        # compacted operands: "staged" (dense copy of the alive rows first, one
        # HBM-bound kvf_stage_rows per compacted level) or "gathered" (TMA gather4
        # of the alive rows straight from the pool, folded units; saves the staging
        # buffer -- U*NB*r bf16 -- but measured 5x slower on the top levels of cfg2:
        # 64 gather4 issues per k-step cannot keep up with the tensor core)
        if compact_mode == "auto":
            compact_mode = "staged"
        if compact_mode not in ("gathered", "staged"):
            raise ConfigError(f"unknown compact_mode {compact_mode!r}")
        if compact_mode == "gathered" and geom.head_mode:
            raise ConfigError("gathered compaction needs folded units")
        self.compact_mode = compact_mode
        self.staged = None
        self.stage_units = U
        if compact_from is not None:
            self.live = torch.empty((U, NB), dtype=torch.int32, device=dev)
            self.rank = torch.empty((U, NB + 1), dtype=torch.int32, device=dev)
            self.acount = torch.empty(U, dtype=torch.int32, device=dev)
            if compact_mode == "staged":
                # staging holds the alive K rows of `stage_units` units at a time (compacted
                # levels run in unit chunks): ~STAGE_BUDGET instead of a second full K pool
                per_unit = NB * geom.r * 2
                self.stage_units = max(1, min(U, stage_budget(self.device) // max(per_unit, 1)))
                self.staged = torch.empty(self.stage_units * NB * geom.r, dtype=torch.bfloat16,
                                          device=dev)

    def capture(self, pool_k: torch.Tensor, pool_v: torch.Tensor, threshold: float, *,
                keep_samples: bool = False) -> "CapturedFusion":
        """Capture run(pool_k, pool_v, threshold) as a CUDA graph (see CapturedFusion).
        The capture itself runs the fusion twice on the pools (warm-up, capture)."""
        return _capture(self, pool_k, pool_v, threshold, keep_samples)

    def run(
        self,
        pool_k: torch.Tensor,
        pool_v: torch.Tensor,
        threshold: float,
        *,
        orig_knorm: torch.Tensor | None = None,
        orig_vnorm: torch.Tensor | None = None,
        table: torch.Tensor | None = None,
        refcount: torch.Tensor | None = None,
        alive: torch.Tensor | None = None,
        keep_samples: bool = False,
        time_sim: bool = False,
        stream=None,
    ) -> FusionState:
        g, dev = self.geom, self.device
        if not -1.0 < threshold < 1.0:
            raise ConfigError(f"threshold must lie strictly inside (-1, 1), got {threshold}")
        if pool_k.dtype != self.dtype or pool_v.dtype != self.dtype:
            raise ConfigError("pool dtype does not match the engine")
        if pool_k.numel() != g.L * g.NB * g.E or pool_v.numel() != pool_k.numel():
            raise ConfigError("pool size does not match the geometry")
        if not (pool_k.is_contiguous() and pool_v.is_contiguous()):
            raise ConfigError("pools must be contiguous")
        sp = N.stream_ptr(stream)
        dt = dtype_code(self.dtype)
        U, NB = g.units, g.NB
        acc = acc_dtype(self.dtype)
        launches = 0
        fuse_knorm = self.fuse_knorm and orig_knorm is None
        if fuse_knorm:  # written by the level-1 similarity launch
            knorm = torch.empty((U, NB), dtype=torch.float32, device=dev)
        else:
            knorm = block_norms(pool_k, g, stream)
            launches += 1
        vnorm = block_norms(pool_v, g, stream)
        launches += 1
        if fuse_knorm:
            oknorm = torch.empty_like(knorm)  # copied from knorm after the level-1 launch
        else:
            oknorm = knorm.clone() if orig_knorm is None else orig_knorm.reshape(U, NB).to(acc)
        ovnorm = vnorm.clone() if orig_vnorm is None else orig_vnorm.reshape(U, NB).to(acc)
        fusable = torch.empty((U, NB), dtype=torch.uint8, device=dev)
        alive_t = torch.empty((U, NB), dtype=torch.uint8, device=dev) if alive is None else alive
        absorber = torch.empty((U, NB), dtype=torch.int32, device=dev)
        table_t = torch.empty((U, NB), dtype=torch.int32, device=dev) if table is None else table
        ref_t = torch.empty((U, NB), dtype=torch.int32, device=dev) if refcount is None else refcount
        N.call(
            "kvf_state_init", dt, U, NB, None if fuse_knorm else N.ptr(oknorm), N.ptr(fusable), N.ptr(alive_t),
            N.ptr(absorber), N.ptr(table_t), N.ptr(ref_t), sp,
        )
        launches += 1
        st = FusionState(
            g, self.plan, threshold, pool_k, pool_v, knorm, vnorm, oknorm, ovnorm, fusable,
            alive_t, absorber, table_t, ref_t,
        )
        st.rescore_cap = self.rescore_cap
        st.path_name = ("simt" if self.path != N.PATH_TC else
                        "tcgen05-split3" if self.filter_mode else "tcgen05")
        st.exact = self.exact or self.filter_mode
        opnd = pool_k  # what the tensor cores read
        if self.filter is not None:
            N.call("kvf_convert_rows", N.ptr(pool_k), dt, N.ptr(self.filter), *g.args(), None, sp)
            opnd = self.filter
            launches += 1
        if self.exact:
            self.sidx.fill_(-1)
            self.scount.zero_()
            st.shadow_count, st.shadow_cap = self.scount, self.shadow_cap
        for li, lv in enumerate(self.levels):
            nm, nt = lv["nm"], lv["nt"]
            stats = torch.empty((U, nm, 8), dtype=torch.float64, device=dev)
            samples = None
            if keep_samples:
                samples = torch.empty((U, max(lv["rect_total"], 1)), dtype=torch.float64, device=dev)
                samples.view(torch.int64).fill_(-1)  # all-ones bit pattern = NaN
            compact = self.compact_from is not None and self.plan.levels[li].height >= self.compact_from
            # compacted levels run in unit chunks that fit the staging buffer
            cu = self.stage_units if compact and self.staged is not None else U
            # re-score band: the fp32 accumulation error at level 1 of a bf16 pool, plus the
            # bf16 rounding of the operands where the tensor cores read rounded copies
            wide = self.exact and self.plan.levels[li].height >= 2
            band = (RESCORE_BAND_WIDE if wide else RESCORE_BAND) if self.rescore_cap else 0.0
            for u0 in range(0, U, cu):
                nU = min(cu, U - u0)
                if compact:
                    N.call("kvf_alive_rank", u0, nU, NB, N.ptr(alive_t), N.ptr(self.live),
                           N.ptr(self.rank), N.ptr(self.acount), sp)
                    launches += 1
                    if self.staged is not None:
                        N.call("kvf_stage_rows", N.ptr(opnd), N.DT_BF16, *g.args(), u0, nU,
                               N.ptr(self.live), N.ptr(self.acount), N.ptr(self.staged), sp)
                        launches += 1
                if time_sim:  # the similarity launch (+ its re-score) only, per chunk
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                N.call(
                    "kvf_similarity_select", N.ptr(pool_k), dt, *g.args(), u0, nU, N.ptr(knorm),
                    N.ptr(fusable), N.ptr(alive_t), N.ptr(absorber), N.ptr(lv["merges"]), nm,
                    # partials are packed per level: unit stride nt * ppt slots of 5 doubles
                    N.ptr(lv["tiles"]), nt, float(threshold),
                    N.ptr(self.partials.view(-1)[u0 * nt * self.ppt * 5:]),
                    N.ptr(samples[u0:]) if samples is not None else None,
                    N.ptr(lv["sample_off"]) if samples is not None else None,
                    samples.shape[1] if samples is not None else 0,
                    N.ptr(self.live) if compact else None, N.ptr(self.rank) if compact else None,
                    N.ptr(self.staged) if compact and self.staged is not None else None,
                    N.ptr(self.rescore), self.rescore_cap, band,
                    N.ptr(self.filter), N.ptr(self.shadow), N.ptr(self.sidx),
                    self.nsplit[li], N.ptr(self.split_part) if self.nsplit[li] > 1 else None,
                    N.ptr(self.split_count) if self.nsplit[li] > 1 else None,
                    (N.PATH_TC_WIDE if self.wide[li] else self.path)
                    | (N.SIM_WRITE_NORMS if fuse_knorm and li == 0 else 0)
                    | (N.SIM_PAIRED if self.paired[li] else 0), sp,
                )
                if self.rescore_cap:
                    launches += 1
                    # pairs within the band of the threshold in this launch (decided in float64)
                    st.near_threshold.append(
                        self.rescore[4 * self.rescore_cap:4 * self.rescore_cap + 1].clone())
                if time_sim:
                    e1.record(stream)
                    st.sim_events.append((e0, e1, li))
            if fuse_knorm and li == 0:  # original key norms = the freshly written ones
                with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
                    oknorm.copy_(knorm)
            N.call(
                "kvf_level_stats", 0, U, U, NB, N.ptr(fusable), N.ptr(alive_t), N.ptr(absorber),
                N.ptr(lv["merges"]), nm, N.ptr(lv["tile_off_p"]), nt * self.ppt,
                N.ptr(self.partials), N.ptr(stats), N.ptr(self.level_ws), sp,
            )
            N.call(
                "kvf_merge_groups", N.ptr(pool_k), N.ptr(pool_v), dt, *g.args(), N.ptr(knorm),
                N.ptr(vnorm), N.ptr(oknorm), N.ptr(ovnorm), N.ptr(self.level_ws),
                3 | (N.MERGE_LAST_LEVEL if li == len(self.levels) - 1 else 0),
                N.ptr(self.shadow), self.shadow_cap, N.ptr(self.sidx), N.ptr(self.scount), sp,
            )
            if self.filter is not None:  # refresh the bf16 copy of the rewritten keys
                N.call("kvf_convert_rows", N.ptr(pool_k), dt, N.ptr(self.filter), *g.args(),
                       N.ptr(self.level_ws), sp)
                launches += 1
            N.call(
                "kvf_remap", 0, U, U, NB, N.ptr(absorber), N.ptr(table_t), N.ptr(ref_t),
                N.ptr(alive_t), N.ptr(self.level_ws), sp,
            )
            launches += 3
            st.level_stats.append(stats)
            st.level_samples.append(samples)
        st.k_scale = torch.empty((U, NB), dtype=acc, device=dev)
        st.v_scale = torch.empty((U, NB), dtype=acc, device=dev)
        st.live_ids = torch.empty((U, NB), dtype=torch.int32, device=dev)
        st.free_ids = torch.empty((U, NB), dtype=torch.int32, device=dev)
        st.live_count = torch.empty(U, dtype=torch.int32, device=dev)
        st.free_count = torch.empty(U, dtype=torch.int32, device=dev)
        N.call(
            "kvf_finalize", dt, 0, U, NB, N.ptr(oknorm), N.ptr(ovnorm), N.ptr(knorm),
            N.ptr(vnorm), N.ptr(table_t), N.ptr(alive_t), N.ptr(st.k_scale), N.ptr(st.v_scale),
            N.ptr(st.live_ids), N.ptr(st.live_count), N.ptr(st.free_ids), N.ptr(st.free_count),
            sp,
        )
        launches += 2
        st.launches = launches
        return st


COMPACT_BIG_MERGE = 65536  # blocks per merge (left + right)
SPLIT_PART_BUDGET = 512 << 20  # bytes of split-K partials per engine
STAGE_BUDGET = 4 << 30  # minimum bytes of staged alive K rows (compacted levels, unit chunks)
STAGE_FREE_FRACTION = 0.25  # ... raised to this share of the free device memory


def stage_budget(device) -> int:
    """Bytes for the staged alive K rows: STAGE_BUDGET, or a quarter of the free device
    memory when that is larger (KVF_STAGE_BUDGET overrides). Every unit chunk of a
    compacted level is one similarity launch with its own last-wave tail, so fewer, larger
    chunks waste less (cfg2: 4 chunks of 8 layers at 4 GB, one chunk of 32 at 16 GB)."""
    env = os.environ.get("KVF_STAGE_BUDGET")
    if env:
        return int(float(env) * (1 << 30))
    budget = STAGE_BUDGET
    try:
        free, _ = torch.cuda.mem_get_info(device)
        budget = max(budget, int(free * STAGE_FREE_FRACTION))
    except Exception:
        pass
    return budget
_TILE_PART_BYTES = 256 * 256 * 4  # one CTA pair's fp32 accumulator tile


# at most 8 k-splits: the last-arriving CTA sums the splits serially (cfg1 per-level similarity
# with max 16 / 8 / 4 / 2 / 1 splits: 0.376 / 0.350 / 0.381 / 0.55 / 0.90 ms per step); KVF_SPLIT_MAX A/B
SPLIT_MAX = int(os.environ.get("KVF_SPLIT_MAX", "8"))


def choose_split(n_tiles: int, nk_run: int, pairs: int) -> int:
    """k-splits per tile for a similarity launch: levels with at most half a wave of
    tiles and long K (folded units: r / 64 k-steps, x3 for float32 hi/lo operands) are
    split so every CTA pair has work; cost model = waves of (tile, split) items x split
    length, +2% per split for the partial write / read-back. Measured: cfg1 (16 / 8 / 4
    tiles, 768 k-steps) similarity 0.93 -> 0.35 ms per step; fuller levels (cfg3 level 1:
    128 tiles, HBM-bound) lose, so they are never split."""
    if n_tiles <= 0 or 2 * n_tiles > pairs or nk_run < 64:
        return 1
    best, best_cost = 1, float(-(-n_tiles // pairs))
    for s in range(2, min(SPLIT_MAX, nk_run // 32) + 1):
        cost = -(-(n_tiles * s) // pairs) / s * (1.0 + 0.02 * s)
        if cost < best_cost - 1e-9:
            best, best_cost = s, cost
    return best


class CapturedFusion:
    """A fusion run captured as one CUDA graph (FusionEngine.capture).

    replay() re-runs every launch of the captured run -- norms, all tree
    levels, finalize -- on the same pool buffers with one host call, removing
    the per-launch host overhead that dominates small caches (CFF chunks).
    The pools are fused in place by every replay, so callers restore them
    first when they need the pristine cache; `state` holds the run's static
    output tensors, overwritten by each replay.
    """

    def __init__(self, graph: torch.cuda.CUDAGraph, state: "FusionState", stream):
        self.graph = graph
        self.state = state
        self.stream = stream

    def replay(self) -> "FusionState":
        self.graph.replay()
        return self.state


def _capture(engine: "FusionEngine", pool_k, pool_v, threshold, keep_samples=False) -> CapturedFusion:
    s = torch.cuda.Stream(engine.device)
    s.wait_stream(torch.cuda.current_stream(engine.device))
    with torch.cuda.stream(s):  # warm-up on the capture stream: per-stream scheduler state,
        engine.run(pool_k, pool_v, threshold, keep_samples=keep_samples)  # kernel attributes
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        st = engine.run(pool_k, pool_v, threshold, keep_samples=keep_samples)
    torch.cuda.current_stream(engine.device).wait_stream(s)
    return CapturedFusion(g, st, s)


def tc_available(geom: Geometry) -> bool:
    """Whether the tcgen05 similarity path accepts this geometry (bf16 pools)."""
    try:
        tile_shape(torch.bfloat16, geom.head_mode, N.PATH_TC)
    except Exception:
        return False
    return _tc_geometry_ok(geom)


def _tc_geometry_ok(geom: Geometry) -> bool:
    # TMA tiles are 64-element (128 B) slices of the head dim
    return geom.d % 64 == 0 and _TC_ENABLED


_TC_ENABLED = True


def audit(table: torch.Tensor, refcount: torch.Tensor, alive: torch.Tensor, U: int, NB: int) -> bool:
    """Device BlockTable.audit (core.py:232-241); True when consistent."""
    scratch = torch.empty(max(U * NB, 1), dtype=torch.int32, device=table.device)
    bad = torch.empty(1, dtype=torch.int32, device=table.device)
    N.call(
        "kvf_table_audit", U, NB, N.ptr(table), N.ptr(refcount), N.ptr(alive), N.ptr(scratch),
        N.ptr(bad), N.stream_ptr(),
    )
    return int(bad.item()) == 0
