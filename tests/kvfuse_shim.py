"""pytest plugin: the reference's own tests against this package -- TEST INFRASTRUCTURE.

Loaded with ``-p kvfuse_shim`` before the reference suite (oracle/_ref_tests, a
git-ignored copy of /root/reference/pkg/tests made by __graft_entry__.build) is
collected. It registers a ``kvfuse`` package whose hot-path modules are this
package's:

    kvfuse.core / kvfuse.fusion / kvfuse.attention / kvfuse.errors
        -> paper_2601_03067_b200.{core, fusion, attention, errors}

while the out-of-scope modules (workload generator, analysis, KVFF I/O, CLI)
load from the installed reference (oracle/_ref/kvfuse) and import the core /
errors they build on from here, i.e. the reference's generator builds this
package's PagedKvCache. Names the hot-path modules do not define (the drift-bound
tools of attention.py, private helpers) are taken from the reference module of
the same name, so ``from kvfuse.attention import verify_drift_bound`` works and
runs the reference's code over this package's caches.
"""

from __future__ import annotations

import importlib.util
import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF_PKG = ROOT / "oracle" / "_ref" / "kvfuse"


def _load_ref_module(name: str) -> types.ModuleType:
    """Execute the reference module `kvfuse.<name>` under a private name."""
    spec = importlib.util.spec_from_file_location(f"kvfuse._ref_{name}", REF_PKG / f"{name}.py")
    mod = importlib.util.module_from_spec(spec)
    mod.__package__ = "kvfuse"
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


def install() -> None:
    if "kvfuse" in sys.modules and getattr(sys.modules["kvfuse"], "__shim__", False):
        return
    if not REF_PKG.exists():
        raise RuntimeError(f"{REF_PKG} missing: run __graft_entry__.build() where /root/reference exists")
    sys.path.insert(0, str(ROOT))
    import paper_2601_03067_b200 as P
    from paper_2601_03067_b200 import attention, core, errors, fusion

    pkg = types.ModuleType("kvfuse")
    pkg.__path__ = [str(REF_PKG)]  # workload / analysis / kvff / cli from the reference
    pkg.__shim__ = True
    sys.modules["kvfuse"] = pkg
    for name, mod in (("errors", errors), ("core", core), ("fusion", fusion), ("attention", attention)):
        sys.modules[f"kvfuse.{name}"] = mod
        setattr(pkg, name, mod)
    # out-of-scope names of the hot-path modules: the reference's definitions, bound
    # to this package's core / errors through the kvfuse.* entries above
    for name, mod in (("core", core), ("fusion", fusion), ("attention", attention)):
        ref = _load_ref_module(name)
        for k, v in vars(ref).items():
            if not k.startswith("__") and not hasattr(mod, k):
                setattr(mod, k, v)
    for k in dir(P):
        if not k.startswith("_"):
            setattr(pkg, k, getattr(P, k))
    import kvfuse.workload  # noqa: F401  (reference generator over this package's core)
    import kvfuse.kvff  # noqa: F401
    import kvfuse.analysis  # noqa: F401

    for k in ("SyntheticSpec", "calibrate_noise", "generate", "generate_fixture"):
        setattr(pkg, k, getattr(sys.modules["kvfuse.workload"], k))
    for k in ("load_cache", "save_cache"):
        setattr(pkg, k, getattr(sys.modules["kvfuse.kvff"], k))


install()
