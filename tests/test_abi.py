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
                                   0, 0.0, None, None, None, 1, None, None, 1, None)
    assert rc == N.KVF_ERR_INVALID
    assert "threshold" in lib.kvf_last_error().decode()
    with pytest.raises(ConfigError):
        N.check(rc)
    rc = lib.kvf_block_norms(None, 2, 0, 1, 1, 1, 1, 0, None, None)
    assert rc == N.KVF_ERR_INVALID
    tm, tn, ppt = C.c_int(), C.c_int(), C.c_int()
    assert lib.kvf_sim_tile_shape(2, 0, N.PATH_TC, C.byref(tm), C.byref(tn), C.byref(ppt)) == 0
    assert (tm.value, tn.value, ppt.value) == (256, 256, 16)  # one moment slot per epilogue warp
    assert lib.kvf_sim_tile_shape(2, 0, N.PATH_TC_WIDE, C.byref(tm), C.byref(tn), C.byref(ppt)) == 0
    assert (tm.value, tn.value, ppt.value) == (512, 256, 16)
    # float32 pools run the tcgen05 path on a bf16 operand copy; float64 pools cannot
    assert lib.kvf_sim_tile_shape(1, 0, N.PATH_TC, C.byref(tm), C.byref(tn), C.byref(ppt)) == 0
    assert lib.kvf_sim_tile_shape(0, 0, N.PATH_TC, C.byref(tm), C.byref(tn), C.byref(ppt)) != 0
    # exact-mode merge / operand copy validate before any CUDA call
    rc = lib.kvf_convert_rows(None, 2, None, 1, 1, 16, 8, 128, 0, None, None)
    assert rc == N.KVF_ERR_INVALID and "float32" in lib.kvf_last_error().decode()
    rc = lib.kvf_merge_groups(None, None, 2, 1, 1, 16, 8, 128, 0, None, None, None, None, None, 3,
                              None, 0, None, None, None)
    assert rc == N.KVF_ERR_INVALID  # null pools
    x = C.c_int()
    p = C.addressof(x)
    rc = lib.kvf_merge_groups(p, p, 1, 1, 1, 16, 8, 128, 0, p, p, p, p, p, 3, p, 1, p, p, None)
    assert rc == N.KVF_ERR_INVALID and "bfloat16" in lib.kvf_last_error().decode()
    rc = lib.kvf_merge_groups(p, p, 2, 1, 1, 16, 8, 128, 0, p, p, p, p, p, 4, None, 0, None, None, None)
    assert rc == N.KVF_ERR_INVALID and "which" in lib.kvf_last_error().decode()


def test_schedule_and_compaction_argument_errors():
    """New entry points validate before touching the GPU."""
    lib = N.lib()
    assert lib.kvf_decode_schedule_item_blocks() in (8, 16)
    # per head unit: block histogram + block reference counts (L2 policy) + item keys
    assert lib.kvf_decode_schedule_ws_ints(0, 8, 1024, 4, 256, 16) == 2 * 1024 + 4 * 16
    assert lib.kvf_decode_schedule_ws_ints(1, 8, 1024, 4, 256, 8) == 8 * 2 * 1024 + 8 * 4 * 32
    assert lib.kvf_decode_schedule_ws_ints(0, 8, 1024, 4, 256, 5) < 0  # bad item size
    # B * p_blocks beyond the layer's slots
    rc = lib.kvf_decode_schedule(None, None, None, 1, 100, 16, 8, 128, 0, 0, 4, 32, None, 16,
                                 None, None, None, None, None, None, None, None, 0, None)
    assert rc == N.KVF_ERR_INVALID and "exceeds" in lib.kvf_last_error().decode()
    # unsupported item size
    rc = lib.kvf_decode_schedule(None, None, None, 1, 1024, 16, 8, 128, 0, 0, 4, 32, None, 12,
                                 None, None, None, None, None, None, None, None, 0, None)
    assert rc == N.KVF_ERR_INVALID and "item_blocks" in lib.kvf_last_error().decode()
    # scheduled decode: probabilities are not offered, GQA group limit
    rc = lib.kvf_paged_decode_sched(None, 2, None, None, 2, 1, 1024, 16, 8, 128, 0, 0, None, None,
                                    None, 4, 32, None, 80, 0.1, None, None, 16, None, None, None,
                                    None, None, 0, None, 1 << 20, None)
    assert rc == N.KVF_ERR_INVALID
    assert lib.kvf_remap_ids(None, -1, None, 0, None, None) == N.KVF_ERR_INVALID
    assert lib.kvf_remap_ids(None, 0, None, 0, None, None) == N.KVF_OK  # empty: nothing to do


def test_similarity_path_flags_validate_before_cuda():
    """Wide tile / paired merges / fused level-1 norms: unsupported combinations are refused
    before any CUDA call (nt = 0, so no device pointer is touched)."""
    lib = N.lib()
    x = C.c_int()
    p = C.addressof(x)

    def sel(dtype, head_mode, nsplit, path, live=None, staged=None, filt=None):
        return lib.kvf_similarity_select(None, dtype, 1, 256, 16, 8, 128, head_mode, 0, 1, None, None,
                                         None, None, None, 0, None, 0, 0.8, None, None, None, 0,
                                         live, live, staged, None, 0, 0.0, filt, None, None, nsplit,
                                         p if nsplit > 1 else None, p if nsplit > 1 else None, path, None)

    rc = sel(2, 0, 2, N.PATH_TC_WIDE)
    assert rc == N.KVF_ERR_INVALID and "nsplit" in lib.kvf_last_error().decode()
    rc = sel(2, 0, 1, N.PATH_TC_WIDE, live=p)  # gathered compaction (no staged rows)
    assert rc == N.KVF_ERR_INVALID and "staged" in lib.kvf_last_error().decode()
    rc = sel(2, 0, 1, N.PATH_TC | N.SIM_PAIRED, live=p, staged=p)
    assert rc == N.KVF_ERR_INVALID and "KVF_SIM_PAIRED" in lib.kvf_last_error().decode()
    rc = sel(2, 0, 1, N.PATH_TC_WIDE | N.SIM_PAIRED)
    assert rc == N.KVF_ERR_INVALID and "KVF_SIM_PAIRED" in lib.kvf_last_error().decode()
    for args in ((1, 0, 1), (2, 0, 2)):  # float32 pool, split-K
        rc = sel(*args, N.PATH_TC | N.SIM_WRITE_NORMS, filt=p if args[0] == 1 else None)
        assert rc == N.KVF_ERR_INVALID and "KVF_SIM_WRITE_NORMS" in lib.kvf_last_error().decode()
    rc = sel(2, 0, 1, N.PATH_TC_WIDE | N.SIM_WRITE_NORMS)
    assert rc == N.KVF_ERR_INVALID and "KVF_SIM_WRITE_NORMS" in lib.kvf_last_error().decode()
