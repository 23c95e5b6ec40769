"""Run only bench.py's decode block (BASELINE configs[3]) and print its JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.set_device(0)
res = bench.bench_decode(torch.device("cuda", 0), torch)
res.pop("cpu_baseline", None)
print(json.dumps(res, indent=1))
