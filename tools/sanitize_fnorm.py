"""Only the level-1 similarity launch with paired merges and fused key norms, for racecheck
(the merge ring's mbarrier-ordered hazards otherwise saturate its hazard counter)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_03067_b200 import _native as N  # noqa: E402
from paper_2601_03067_b200.engine import FusionEngine, Geometry, block_norms  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

Kt, Vt = synthetic_kv(2, 16, 64, 16, 8, 128, dtype=torch.bfloat16, seed=12)
geom = Geometry(2, 16 * 64, 16, 8, 128, 0)
eng = FusionEngine(geom, bff_plan(16, 64, None), torch.bfloat16, Kt.device, split=False)
assert eng.paired[0] and eng.fuse_knorm
# one fusion run, but stop after level 1 by running the engine with a one-level plan copy
plan1 = bff_plan(16, 64, None)
plan1.levels = plan1.levels[:1]
eng1 = FusionEngine(geom, plan1, torch.bfloat16, Kt.device, split=False, compact_from=None)
assert eng1.paired[0] and eng1.fuse_knorm
st = eng1.run(Kt.reshape(-1).clone(), Vt.reshape(-1).clone(), 0.8)
torch.cuda.synchronize()
ref = block_norms(Kt.reshape(-1).contiguous(), geom)
print("level-1 fused norms max rel diff", float(((st.orig_knorm - ref).abs() / ref).max()))
