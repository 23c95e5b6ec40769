import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


@lru_cache(maxsize=1)
def golden():
    arrays = dict(np.load(GOLDEN / "golden.npz"))
    meta = json.loads((GOLDEN / "golden.json").read_text())
    return arrays, meta


def golden_cases(kind=None):
    _, meta = golden()
    return [c for c in meta["cases"] if kind is None or c["kind"] in (kind if isinstance(kind, tuple) else (kind,))]


def unit_inputs(case):
    """(kflat, vflat, rows, bpr, groups_kind) for a golden case."""
    arrays, _ = golden()
    kind = case["kind"]
    if kind == "fast_fusion_fixture":
        k = arrays[f"fixture/{case['fixture']}/keys"][case["layer"]]
        v = arrays[f"fixture/{case['fixture']}/values"][case["layer"]]
        B, p = k.shape[:2]
        return k.reshape(B * p, -1), v.reshape(B * p, -1), B, p
    if kind == "fast_fusion_rows":
        k = arrays[f"rows/{case['seed']}/k"]
        v = arrays[f"rows/{case['seed']}/v"]
        return k.reshape(-1, k.shape[-1]), v.reshape(-1, v.shape[-1]), k.shape[0], k.shape[1]
    if kind == "hand":
        a = arrays[f"hand/{case['hname']}/rows"]
        return a.reshape(-1, a.shape[-1]), a.reshape(-1, a.shape[-1]), a.shape[0], a.shape[1]
    raise KeyError(kind)


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
