import sys, torch
sys.path.insert(0, '.')
from paper_2601_03067_b200.engine import FusionEngine, Geometry, stage_budget
from paper_2601_03067_b200.schedule import bff_plan
dev = torch.device('cuda', 0)
x = torch.empty(4 * 8589934592, dtype=torch.bfloat16, device=dev)  # 68.7 GB like the bench pools
print('free', torch.cuda.mem_get_info(dev), 'budget', stage_budget(dev))
eng = FusionEngine(Geometry(32, 16384, 16, 8, 128, 0), bff_plan(64, 256, None), torch.bfloat16, dev)
print('stage_units', eng.stage_units, 'wide', eng.wide, 'free after', torch.cuda.mem_get_info(dev))
