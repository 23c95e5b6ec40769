"""ctypes binding of libkvfuse_b200.so (include/kvfuse_b200.h).

The library is the product path: there is no CPU or eager-PyTorch fallback.
If it is missing, `lib()` raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import AlignmentError, ConfigError, CorruptionError, KvFuseError

LIB_PATH = Path(
    os.environ.get("KVF_LIB") or Path(__file__).resolve().parent / "_lib" / "libkvfuse_b200.so"
)  # KVF_LIB: load another build of the library (A/B measurements)

KVF_OK = 0
KVF_ERR_INVALID = 1
KVF_ERR_ALIGNMENT = 2
KVF_ERR_CORRUPTION = 3
KVF_ERR_CUDA = 4

PATH_AUTO = 0
PATH_SIMT = 1
PATH_TC = 2
PATH_TC_WIDE = 3  # tcgen05, 512 x 256 tile per CTA pair
SIM_WRITE_NORMS = 0x100  # OR-ed into the path: level-1 launch computes the key norms
SIM_PAIRED = 0x200  # OR-ed into the path: two small merges per tile (diagonal)
MERGE_LAST_LEVEL = 0x10  # OR-ed into kvf_merge_groups' which: shadow rows read, not written

DT_F64, DT_F32, DT_BF16 = 0, 1, 2

_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_f64 = C.c_double

# name -> (restype, argtypes); mirrors include/kvfuse_b200.h
SIGNATURES: dict[str, tuple] = {
    "kvf_last_error": (C.c_char_p, []),
    "kvf_version": (_i32, []),
    "kvf_count_nonfinite": (_i32, [_vp, _i32, _i64, _vp, _vp]),
    "kvf_block_norms": (_i32, [_vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _vp, _vp]),
    "kvf_state_init": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kvf_sim_tile_shape": (
        _i32, [_i32, _i32, _i32, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]
    ),
    "kvf_similarity_select": (
        _i32,
        [_vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _i64, _i64, _vp, _vp, _vp, _vp,
         _vp, _i32, _vp, _i32, _f64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _f64,
         _vp, _vp, _vp, _i32, _vp, _vp, _i32, _vp],
    ),
    "kvf_convert_rows": (_i32, [_vp, _i32, _vp, _i64, _i64, _i32, _i32, _i32, _i32, _vp, _vp]),
    "kvf_alive_rank": (_i32, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "kvf_stage_rows": (
        _i32, [_vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _i64, _i64, _vp, _vp, _vp, _vp]
    ),
    "kvf_level_ws_ints": (_i64, [_i64]),
    "kvf_level_stats": (
        _i32,
        [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp],
    ),
    "kvf_merge_groups": (
        _i32, [_vp, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i32,
               _vp, _i64, _vp, _vp, _vp]
    ),
    "kvf_remap": (_i32, [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kvf_finalize": (
        _i32,
        [_i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
         _vp],
    ),
    "kvf_table_audit": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kvf_table_redirect": (_i32, [_i64, _vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "kvf_gather_vectors": (
        _i32, [_vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _i64, _vp, _i64, _vp, _vp, _vp, _vp]
    ),
    "kvf_refold": (
        _i32, [_vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _i64, _vp, _vp, _vp, _vp]
    ),
    "kvf_decode_workspace_size": (_i64, [_i32, _i64, _i32, _i32, _i64, _i32]),
    "kvf_paged_decode": (
        _i32,
        [_vp, _i32, _vp, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _i64, _vp, _vp, _vp,
         _i64, _i64, _vp, _i32, _f64, _vp, _vp, _vp, _vp, _i64, _vp],
    ),
    "kvf_remap_ids": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp]),
    "kvf_chunk_prefill": (
        _i32,
        [_vp, _vp, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _i64, _vp, _vp, _vp, _vp, _i64,
         _i64, _i32, _i32, _i32, _f64, _i32, _i32, _vp, _vp],
    ),
    "kvf_quantile_ws_bytes": (_i64, []),
    "kvf_quantile": (_i32, [_vp, _vp, _i32, _f64, _vp, _vp, _i64, _vp]),
    "kvf_decode_schedule_item_blocks": (_i32, []),
    "kvf_decode_schedule_ws_ints": (_i64, [_i32, _i32, _i64, _i64, _i64, _i32]),
    "kvf_decode_schedule": (
        _i32,
        [_vp, _vp, _vp, _i64, _i64, _i32, _i32, _i32, _i32, _i64, _i64, _i64, _vp, _i32, _vp,
         _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp],
    ),
    "kvf_paged_decode_sched": (
        _i32,
        [_vp, _i32, _vp, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _i32, _i64, _vp, _vp, _vp,
         _i64, _i64, _vp, _i32, _f64, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _i64,
         _vp],
    ),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


class NativeLibraryError(KvFuseError):
    """The CUDA extension is missing or failed to load."""


class CudaError(KvFuseError):
    """A CUDA launch / runtime failure reported by the library."""


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing; run `python -m paper_2601_03067_b200.build` "
                    "(there is no CPU fallback)"
                )
            handle = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(rc: int, exc: type[KvFuseError] | None = None) -> None:
    """Map a C status code to the reference's exception classes (errors.py)."""
    if rc == KVF_OK:
        return
    msg = lib().kvf_last_error().decode(errors="replace")
    if exc is not None:
        raise exc(msg)
    if rc == KVF_ERR_INVALID:
        raise ConfigError(msg)
    if rc == KVF_ERR_ALIGNMENT:
        raise AlignmentError(msg)
    if rc == KVF_ERR_CORRUPTION:
        raise CorruptionError(msg)
    raise CudaError(msg)


def call(name: str, *args, exc: type[KvFuseError] | None = None) -> None:
    check(getattr(lib(), name)(*args), exc)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
