"""Run only bench.py's adaptive-threshold block and print its JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.set_device(0)
print(json.dumps(bench.bench_adaptive_threshold(torch.device("cuda", 0), torch), indent=1))
