"""Host-side fusion schedule: the data-independent shape of the merge tree.

The reference recursion (fusion.py:230-240) splits a row list at
``mid = len // 2`` and merges the two halves after both are fused; its height
is ``max(dl, dr) + 1``. Independent trees come from ``_grouped``
(fusion.py:354-357) and, for CFF, from the per-request row ranges
(fusion.py:404-407). Because survivor lists stay in ascending block-id order
(fusion.py:282), every merge node owns a contiguous row range and its alive
blocks are exactly the alive blocks of that range. Merges of equal height are
independent, so the device runs the tree level by level (one launch set per
height) instead of recursively.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np


def grouped(indices: list[int], group_size: int | None) -> list[list[int]]:
    """Consecutive row groups (fusion.py:354-357)."""
    if group_size is None or group_size >= len(indices):
        return [list(indices)]
    return [list(indices[i : i + group_size]) for i in range(0, len(indices), group_size)]


# tile rows per launch-order band (L2 reuse of operand tiles); KVF_TILE_BAND overrides (A/B)
TILE_BAND = int(os.environ.get("KVF_TILE_BAND", "4"))


@dataclass(frozen=True)
class MergeNode:
    height: int
    row_lo: int
    row_mid: int
    row_hi: int
    post: int  # index in the reference's _merge call order (post-order)


def _tree(lo: int, hi: int, nodes: list[MergeNode]) -> int:
    """Recursion of fusion.py:230-240 over rows [lo, hi); returns height."""
    n = hi - lo
    if n == 1:
        return 0
    mid = lo + n // 2
    dl = _tree(lo, mid, nodes)
    dr = _tree(mid, hi, nodes)
    height = max(dl, dr) + 1
    nodes.append(MergeNode(height, lo, mid, hi, len(nodes)))
    return height


@dataclass
class Level:
    height: int
    nodes: list[MergeNode]
    merges: np.ndarray  # int32 [nm, 3] block ranges (left_begin, split, right_end)
    post: np.ndarray  # int32 [nm]
    row_merge: np.ndarray  # int32 [rows], merge index of the row at this level or -1
    tiles: dict = field(default_factory=dict)  # (tm, tn) -> (tiles [nt,3], tile_off [nm+1])

    def tiling(self, tm: int, tn: int, band: int = TILE_BAND) -> tuple[np.ndarray, np.ndarray]:
        """Tiles (merge, i0, j0) of every merge, launch-ordered in bands of
        `band` tile rows walked column by column, so CTAs running together
        share A and B operand rows in L2."""
        key = (tm, tn, band)
        if key not in self.tiles:
            tl, off = [], [0]
            for m, (lb, mid, re) in enumerate(self.merges.tolist()):
                rows = list(range(0, mid - lb, tm))
                cols = list(range(0, re - mid, tn))
                for b0 in range(0, len(rows), band):
                    for j0 in cols:
                        for i0 in rows[b0 : b0 + band]:
                            tl.append((m, i0, j0))
                off.append(len(tl))
            self.tiles[key] = (
                np.asarray(tl, dtype=np.int32).reshape(-1, 3),
                np.asarray(off, dtype=np.int32),
            )
        return self.tiles[key]

    def rect_sizes(self) -> np.ndarray:
        lb, mid, re = self.merges[:, 0], self.merges[:, 1], self.merges[:, 2]
        return (mid - lb).astype(np.int64) * (re - mid).astype(np.int64)


@dataclass
class Plan:
    """Merge schedule for one unit structure (shared by all layers / heads)."""

    rows: int
    bpr: int
    groups: list[tuple[int, int]]
    levels: list[Level]
    merge_calls: int
    tree_depth: int
    nodes: list[MergeNode]  # in post-order

    @property
    def n_blocks(self) -> int:
        return self.rows * self.bpr


def build_plan(rows: int, bpr: int, groups: list[list[int]]) -> Plan:
    nodes: list[MergeNode] = []
    ranges: list[tuple[int, int]] = []
    depth = 0
    for grp in groups:
        lo, hi = grp[0], grp[-1] + 1
        if list(grp) != list(range(lo, hi)):
            raise ValueError("row groups must be contiguous ranges")
        ranges.append((lo, hi))
        sub: list[MergeNode] = []
        d = _tree(lo, hi, sub)
        base = len(nodes)
        nodes.extend(MergeNode(n.height, n.row_lo, n.row_mid, n.row_hi, base + n.post) for n in sub)
        depth = max(depth, d)
    levels = []
    for hgt in range(1, depth + 1):
        lv = [n for n in nodes if n.height == hgt]
        merges = np.asarray(
            [(n.row_lo * bpr, n.row_mid * bpr, n.row_hi * bpr) for n in lv], dtype=np.int32
        ).reshape(-1, 3)
        row_merge = np.full(rows, -1, dtype=np.int32)
        for m, n in enumerate(lv):
            row_merge[n.row_lo : n.row_hi] = m
        levels.append(
            Level(hgt, lv, merges, np.asarray([n.post for n in lv], dtype=np.int32), row_merge)
        )
    return Plan(rows, bpr, ranges, levels, len(nodes), depth, nodes)


def bff_plan(B: int, p: int, group_size: int | None) -> Plan:
    """BFF rows = requests (fusion.py:367-370)."""
    return build_plan(B, p, grouped(list(range(B)), group_size))


def cff_plan(B: int, C: int, blocks_per_chunk: int, group_size: int | None) -> Plan:
    """CFF rows = (request, chunk); trees never cross requests (fusion.py:404-407)."""
    groups: list[list[int]] = []
    for req in range(B):
        groups.extend(grouped(list(range(req * C, (req + 1) * C)), group_size))
    return build_plan(B * C, blocks_per_chunk, groups)


def single_tree_plan(rows: int, bpr: int) -> Plan:
    """fast_fusion: one tree over all rows (fusion.py:348-350)."""
    return build_plan(rows, bpr, [list(range(rows))])
