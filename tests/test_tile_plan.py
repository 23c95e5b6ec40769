"""Host-side choice of the similarity launch per tree level (engine.tile_plan): paired small
merges, split-K, the wide 512 x 256 tile, compaction and the fused level-1 key norms, for
every BASELINE configuration (no GPU: the plan is pure host logic over the tree)."""

import torch

from paper_2601_03067_b200 import _native as N
from paper_2601_03067_b200.core import cff_layout
from paper_2601_03067_b200.engine import Geometry, tile_plan
from paper_2601_03067_b200.schedule import bff_plan, cff_plan

PAIRS = 74  # CTA pairs of a B200 (148 SMs)


def _plan(L, B, p, head_mode=0, dtype=torch.bfloat16, variant="bff", env=None, split=True):
    t, h, d = 16, 8, 128
    if variant == "cff":
        C, bpc = cff_layout(p, t, 2048)
        plan = cff_plan(B, C, bpc, None)
    else:
        plan = bff_plan(B, p, None)
    return tile_plan(plan, Geometry(L, B * p, t, h, d, head_mode), dtype, N.PATH_TC, "auto", "staged",
                     split, PAIRS, env=env or {})


def test_cfg2_folded():
    tp = _plan(32, 64, 256)
    assert tp.compact_from == 5
    assert tp.wide == [False, True, True, True, True, True]  # level 1: 256-block merges
    assert tp.paired == [False] * 6 and tp.nsplit == [1] * 6
    assert tp.fuse_knorm  # every block is an operand row of exactly one level-1 tile


def test_cfg2_shard_of_8_gpus():
    tp = _plan(4, 64, 256)  # 4 layers per rank at N = 8
    assert tp.wide == [False, False, True, True, True, True]  # level 2: one wave of wide tiles
    assert tp.fuse_knorm


def test_cfg2_per_head():
    tp = _plan(32, 64, 256, head_mode=1)
    assert not any(tp.wide)  # short-K tiles keep the double-buffered accumulator
    assert tp.fuse_knorm and tp.compact_from == 5


def test_cfg3_cff():
    tp = _plan(32, 1, 1024, variant="cff")
    assert tp.paired == [True, False, False]  # 128 x 128 chunk merges, two per tile
    assert tp.compact_from is None and tp.fuse_knorm
    assert tp.nt[0] == 2  # 4 merges per unit -> 2 paired tiles


def test_cfg1_float32():
    tp = _plan(4, 8, 64, dtype=torch.float32)
    assert tp.paired == [True, True, False]
    assert max(tp.nsplit) > 1 and not any(tp.wide)
    assert not tp.fuse_knorm and tp.compact_from is None  # hi / lo operand copy


def test_cfg5_layer():
    tp = _plan(1, 256, 1024)
    assert tp.compact_from == 6  # depth 8; the 65,536-block merges compact one level lower
    assert all(tp.wide)
    assert not tp.fuse_knorm  # level-1 merges span 1,024 blocks: several tiles per row


def test_env_knobs():
    assert not any(_plan(32, 64, 256, env={"KVF_SIM_WIDE": "0"}).wide)
    assert not any(_plan(32, 1, 1024, variant="cff", env={"KVF_SIM_PAIRED": "0"}).paired)
    assert not _plan(32, 64, 256, env={"KVF_FUSE_KNORM": "0"}).fuse_knorm
    tp = _plan(2, 16, 96, env={"KVF_SIM_WIDE": "1"}, split=False)
    assert all(w or p for w, p in zip(tp.wide, tp.paired))
