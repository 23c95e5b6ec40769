"""CPU checks of the C ABI boundary: the library loads, exports every entry
point include/kvfuse_b200.h declares, the ctypes signature table covers
them, and argument validation maps to the reference's exception classes
without touching a GPU."""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2601_03067_b200 import _native as N
from paper_2601_03067_b200.errors import ConfigError

HEADER = Path(__file__).resolve().parent.parent / "include" / "kvfuse_b200.h"


def _declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kvf_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("kvf_block_norms", "kvf_similarity_select", "kvf_merge_groups", "kvf_remap",
                 "kvf_paged_decode", "kvf_last_error", "kvf_finalize", "kvf_level_stats"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in _declared():
        assert hasattr(lib, name), name


def test_ctypes_table_matches_header():
    assert sorted(N.SIGNATURES) == _declared()


def test_argument_errors_map_to_reference_exceptions():
    lib = N.lib()
    # invalid threshold / dims are rejected before any CUDA call
    rc = lib.kvf_similarity_select(None, 2, 1, 1, 1, 1, 64, 0, 0, 1, None, None, None, None, None,
                                   0, None, 0, 1.5, None, None, None, 0, None, None, None, None,
                                   0, 0.0, 1, None)
    assert rc == N.KVF_ERR_INVALID
    assert "threshold" in lib.kvf_last_error().decode()
    with pytest.raises(ConfigError):
        N.check(rc)
    rc = lib.kvf_block_norms(None, 2, 0, 1, 1, 1, 1, 0, None, None)
    assert rc == N.KVF_ERR_INVALID
    tm, tn, ppt = C.c_int(), C.c_int(), C.c_int()
    assert lib.kvf_sim_tile_shape(2, 0, N.PATH_TC, C.byref(tm), C.byref(tn), C.byref(ppt)) == 0
    assert (tm.value, tn.value, ppt.value) == (256, 256, 2)
    assert lib.kvf_sim_tile_shape(1, 0, N.PATH_TC, C.byref(tm), C.byref(tn), C.byref(ppt)) != 0
