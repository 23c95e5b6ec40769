"""Paged KV-cache model, block tables and the fused-cache containers.

Drop-in counterparts of the reference's kvfuse.core (core.py:1-305) with the
same names, attributes and error behaviour, but device resident: cache tensors
live in HBM (torch CUDA storage), block tables are int32 device arrays updated
by the library's remap kernels, and `refold` gathers through the table on the
GPU. Host-facing attributes (`entries`, `refcount`, `directions`, LayerView
arrays) are materialised lazily for API parity.
"""

from __future__ import annotations

from collections.abc import MutableMapping
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .engine import Geometry, acc_dtype, block_norms, dtype_code
from .errors import AlignmentError, CorruptionError, InvalidCacheError, ZeroVectorError

DIRECTION_NORM_TOL = 1e-5


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise N.NativeLibraryError("a CUDA device is required (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class CacheDims:
    """Dimensions of a paged cache (core.py:23-51)."""

    B: int
    p: int
    t: int
    h: int
    d: int
    L: int

    def __post_init__(self):
        for name in ("B", "p", "t", "h", "d", "L"):
            value = getattr(self, name)
            if isinstance(value, bool) or not isinstance(value, (int, np.integer)) or value < 1:
                raise InvalidCacheError(f"dimension {name} must be a positive integer, got {value!r}")

    @property
    def r(self) -> int:
        return self.t * self.h * self.d

    @property
    def tokens_per_request(self) -> int:
        return self.p * self.t

    @property
    def shape(self) -> tuple[int, ...]:
        return (self.L, self.B, self.p, self.t, self.h, self.d)


def _count_nonfinite(t: torch.Tensor) -> int:
    cnt = torch.zeros(1, dtype=torch.int64, device=t.device)
    N.call("kvf_count_nonfinite", N.ptr(t), dtype_code(t.dtype), t.numel(), N.ptr(cnt), N.stream_ptr())
    return int(cnt.item())


class PagedKvCache:
    """K/V tensors in the paged (L, B, p, t, h, d) layout (core.py:54-76).

    numpy inputs are widened to float64 exactly like the reference and
    mirrored to the GPU (``keys_dev`` / ``values_dev``); torch CUDA tensors
    (float64 / float32 / bfloat16) are used in place without a host copy.
    NaN / Inf entries raise InvalidCacheError (checked on the device).

    ``defer_upload=True`` with host (ideally pinned) torch tensors keeps the
    cache on the host: fuse_batch / fuse_chunks then stream it to the GPU in
    layer chunks overlapped with fusion, validating each chunk on the device
    (a non-finite entry raises InvalidCacheError from the fuse call).
    """

    def __init__(self, dims: CacheDims, keys, values, *, defer_upload: bool = False):
        self.dims = dims
        self.keys_dev = self.values_dev = None
        if (defer_upload and isinstance(keys, torch.Tensor) and isinstance(values, torch.Tensor)
                and not keys.is_cuda and not values.is_cuda):
            if tuple(keys.shape) != dims.shape or tuple(values.shape) != dims.shape:
                raise InvalidCacheError(f"keys / values shapes do not match dims {dims.shape}")
            if keys.dtype != values.dtype or keys.dtype not in (torch.float32, torch.bfloat16):
                raise InvalidCacheError("deferred upload takes float32 or bfloat16 host tensors")
            self.keys = keys.contiguous()
            self.values = values.contiguous()
            self._device = default_device()
            return
        if isinstance(keys, torch.Tensor) or isinstance(values, torch.Tensor):
            if not (isinstance(keys, torch.Tensor) and isinstance(values, torch.Tensor)):
                raise InvalidCacheError("keys and values must both be torch tensors or arrays")
            if tuple(keys.shape) != dims.shape:
                raise InvalidCacheError(f"keys shape {tuple(keys.shape)} does not match dims {dims.shape}")
            if tuple(values.shape) != tuple(keys.shape):
                raise InvalidCacheError(
                    f"values shape {tuple(values.shape)} differs from keys shape {tuple(keys.shape)}"
                )
            if keys.dtype != values.dtype:
                raise InvalidCacheError("keys and values must share a dtype")
            dev = keys.device if keys.is_cuda else default_device()
            kd = keys.to(dev).contiguous()
            vd = values.to(dev).contiguous()
            if kd.dtype not in (torch.float64, torch.float32, torch.bfloat16):
                kd, vd = kd.double(), vd.double()
            self.keys = kd
            self.values = vd
        else:
            k = np.asarray(keys, dtype=np.float64)
            v = np.asarray(values, dtype=np.float64)
            if k.shape != dims.shape:
                raise InvalidCacheError(f"keys shape {k.shape} does not match dims {dims.shape}")
            if v.shape != k.shape:
                raise InvalidCacheError(f"values shape {v.shape} differs from keys shape {k.shape}")
            self.keys = k
            self.values = v
            dev = default_device()
            kd = torch.from_numpy(np.ascontiguousarray(k)).to(dev)
            vd = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
        if _count_nonfinite(kd) or _count_nonfinite(vd):
            raise InvalidCacheError("cache contains NaN or Inf entries")
        self.keys_dev = kd
        self.values_dev = vd
        self._device = kd.device

    @property
    def host_resident(self) -> bool:
        """True while a deferred-upload cache has not been copied to the GPU."""
        return self.keys_dev is None

    @property
    def dtype(self) -> torch.dtype:
        return self.keys.dtype if self.keys_dev is None else self.keys_dev.dtype

    @property
    def device(self) -> torch.device:
        return self._device

    def geometry(self, head_mode: int = 0) -> Geometry:
        d = self.dims
        return Geometry(d.L, d.B * d.p, d.t, d.h, d.d, head_mode)


class UnfoldedLayer:
    """Unit directions (rows, blocks_per_row, r) + norms (core.py:79-112).

    Accepts numpy arrays (reference semantics) or torch tensors.
    """

    def __init__(self, vectors, norms):
        self.vectors = vectors
        self.norms = norms
        vs, ns = tuple(vectors.shape), tuple(norms.shape)
        if len(vs) != 3 or ns != vs[:2]:
            raise InvalidCacheError(f"inconsistent unfolded shapes {vs} / {ns}")

    @property
    def rows(self) -> int:
        return self.vectors.shape[0]

    @property
    def blocks_per_row(self) -> int:
        return self.vectors.shape[1]

    @property
    def r(self) -> int:
        return self.vectors.shape[2]

    @property
    def fusable(self):
        return self.norms > 0.0


def _to_np(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _unfold_unit_rows(cache: PagedKvCache, layer: int, rows: int, bpr: int, req: int | None):
    """Directions + norms of one layer (or one request of it) via K1 + gather."""
    g = cache.geometry(0)
    out = []
    for pool in (cache.keys_dev, cache.values_dev):
        full_norms = block_norms(pool, g)
        norms = full_norms[layer]  # [NB]
        if req is None:
            ids = torch.arange(g.NB, dtype=torch.int32, device=pool.device)
        else:
            ids = torch.arange(req * cache.dims.p, (req + 1) * cache.dims.p, dtype=torch.int32, device=pool.device)
        dirs = torch.empty((ids.numel(), g.r), dtype=acc_dtype(pool.dtype), device=pool.device)
        N.call(
            "kvf_gather_vectors", N.ptr(pool), dtype_code(pool.dtype), *g.args(), layer, N.ptr(ids),
            ids.numel(), N.ptr(full_norms), None, N.ptr(dirs), N.stream_ptr(),
        )
        nrm = norms[ids.long()]
        out.append(
            UnfoldedLayer(
                _to_np(dirs).astype(np.float64).reshape(rows, bpr, g.r),
                _to_np(nrm).astype(np.float64).reshape(rows, bpr),
            )
        )
    return out[0], out[1]


def unfold_bff(cache: PagedKvCache, layer: int) -> tuple[UnfoldedLayer, UnfoldedLayer]:
    """Per-request (B, p, r) unfolding of one layer (core.py:122-131)."""
    if not 0 <= layer < cache.dims.L:
        raise InvalidCacheError(f"layer {layer} out of range [0, {cache.dims.L})")
    return _unfold_unit_rows(cache, layer, cache.dims.B, cache.dims.p, None)


def cff_chunk_count(p: int, t: int, chunk_tokens: int) -> int:
    """C = (p*t) // chunk_tokens with the reference's checks (core.py:134-140)."""
    if chunk_tokens < 1 or chunk_tokens % t != 0:
        raise AlignmentError(f"chunk_tokens={chunk_tokens} is not a positive multiple of t={t}")
    if chunk_tokens > p * t:
        raise AlignmentError(f"chunk_tokens={chunk_tokens} exceeds the request's {p * t} tokens")
    return (p * t) // chunk_tokens


def cff_layout(p: int, t: int, chunk_tokens: int) -> tuple[int, int]:
    C = cff_chunk_count(p, t, chunk_tokens)
    if p % C != 0:
        raise AlignmentError(f"chunk count C={C} does not divide p={p}; blocks cannot be split evenly")
    return C, p // C


def unfold_cff(cache: PagedKvCache, layer: int, chunk_tokens: int, request: int = 0):
    """Per-chunk (C, p/C, r) unfolding of one request (core.py:143-161)."""
    if not 0 <= layer < cache.dims.L:
        raise InvalidCacheError(f"layer {layer} out of range [0, {cache.dims.L})")
    if not 0 <= request < cache.dims.B:
        raise InvalidCacheError(f"request {request} out of range [0, {cache.dims.B})")
    C, bpc = cff_layout(cache.dims.p, cache.dims.t, chunk_tokens)
    return _unfold_unit_rows(cache, layer, C, bpc, request)


def cosine_similarity(a, b) -> float:
    """Cosine of two host vectors, clamped to [-1, 1] (core.py:164-172).

    A scalar utility on host values; not part of the fusion path.
    """
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    na = float(np.sqrt(np.dot(a, a)))
    nb = float(np.sqrt(np.dot(b, b)))
    if na == 0.0 or nb == 0.0:
        raise ZeroVectorError("cosine similarity undefined for a zero vector")
    return float(np.clip(np.dot(a, b) / (na * nb), -1.0, 1.0))


Slot = tuple[int, int]


class _RefcountView(MutableMapping):
    """dict-like view {live phys: refcount} over device arrays (write-through)."""

    def __init__(self, table: "BlockTable"):
        self._t = table

    def _host(self):
        return self._t._host_state()

    def __getitem__(self, phys):
        alive, ref, _ = self._host()
        if not (0 <= phys < alive.size) or not alive[phys]:
            raise KeyError(phys)
        return int(ref[phys])

    def __setitem__(self, phys, value):
        self._t._refcount[int(phys)] = int(value)
        self._t._mutated()

    def __delitem__(self, phys):
        alive, _, _ = self._host()
        if not alive[phys]:
            raise KeyError(phys)
        self._t._refcount[int(phys)] = 0
        self._t._alive[int(phys)] = 0
        self._t._mutated()

    def __iter__(self):
        alive, _, _ = self._host()
        return iter(int(i) for i in np.nonzero(alive)[0])

    def __len__(self):
        alive, _, _ = self._host()
        return int(alive.sum())

    def pop(self, phys, *default):
        try:
            v = self[phys]
        except KeyError:
            if default:
                return default[0]
            raise
        del self[phys]
        return v


class _EntriesView(MutableMapping):
    """dict-like view {(row, blk): phys} over the device table (write-through)."""

    def __init__(self, table: "BlockTable"):
        self._t = table

    def __getitem__(self, slot):
        i, j = slot
        if not (0 <= i < self._t.rows and 0 <= j < self._t.blocks_per_row):
            raise KeyError(slot)
        _, _, tab = self._t._host_state()
        return int(tab[i * self._t.blocks_per_row + j])

    def __setitem__(self, slot, phys):
        i, j = slot
        self._t._table[i * self._t.blocks_per_row + j] = int(phys)
        self._t._mutated()

    def __delitem__(self, slot):
        raise CorruptionError("logical slots cannot be removed from a paged block table")

    def __iter__(self):
        bpr = self._t.blocks_per_row
        return iter((s // bpr, s % bpr) for s in range(self._t.rows * bpr))

    def __len__(self):
        return self._t.rows * self._t.blocks_per_row

    def items(self):
        _, _, tab = self._t._host_state()
        bpr = self._t.blocks_per_row
        return [((s // bpr, s % bpr), int(p)) for s, p in enumerate(tab.tolist())]


class BlockTable:
    """Per-unit logical slot -> physical block map with refcounts (core.py:178-241).

    Storage is three int32/uint8 device arrays of length rows*blocks_per_row
    (slot -> phys table, per-block refcount, per-block alive flag); the
    reference's dicts are exposed as write-through views.
    """

    def __init__(self, layer: int, rows: int, blocks_per_row: int, table: torch.Tensor,
                 refcount: torch.Tensor, alive: torch.Tensor):
        self.layer = layer
        self.rows = rows
        self.blocks_per_row = blocks_per_row
        self._table = table
        self._refcount = refcount
        self._alive = alive
        self.reusable: set[int] = set()
        self._cache = None
        self._listeners: list = []  # called after a mutation (derived per-slot scales)

    @classmethod
    def identity(cls, layer: int, rows: int, blocks_per_row: int, device=None) -> "BlockTable":
        dev = device or default_device()
        n = rows * blocks_per_row
        return cls(
            layer, rows, blocks_per_row,
            torch.arange(n, dtype=torch.int32, device=dev),
            torch.ones(n, dtype=torch.int32, device=dev),
            torch.ones(n, dtype=torch.uint8, device=dev),
        )

    # -- host mirror -------------------------------------------------------
    def _dirty(self):
        self._cache = None

    def _mutated(self):
        """A slot or refcount changed (redirect, entries / refcount writes): drop the
        host mirror and let dependents (the fused unit's per-slot K / V scales,
        K_s = key_norm[s] / |x_table[s]| * x_table[s]) recompute on the device."""
        self._cache = None
        for fn in self._listeners:
            fn()

    def _host_state(self):
        if self._cache is None:
            self._cache = (
                self._alive.cpu().numpy().astype(bool),
                self._refcount.cpu().numpy(),
                self._table.cpu().numpy(),
            )
        return self._cache

    @property
    def entries(self) -> _EntriesView:
        return _EntriesView(self)

    @property
    def refcount(self) -> _RefcountView:
        return _RefcountView(self)

    @property
    def _slots(self) -> dict[int, set[Slot]]:
        _, _, tab = self._host_state()
        out: dict[int, set[Slot]] = {}
        bpr = self.blocks_per_row
        for s, p in enumerate(tab.tolist()):
            out.setdefault(int(p), set()).add((s // bpr, s % bpr))
        return out

    @property
    def device_table(self) -> torch.Tensor:
        return self._table

    @property
    def device_refcount(self) -> torch.Tensor:
        return self._refcount

    @property
    def device_alive(self) -> torch.Tensor:
        return self._alive

    # -- reference API -----------------------------------------------------
    def physical_of(self, slot: Slot) -> int:
        try:
            return self.entries[slot]
        except (KeyError, TypeError, ValueError):
            raise CorruptionError(f"unknown logical slot {slot}") from None

    def is_shared(self, slot: Slot) -> bool:
        return self.refcount[self.physical_of(slot)] > 1

    def slots_of(self, phys: int) -> frozenset[Slot]:
        alive, _, tab = self._host_state()
        if not (0 <= phys < alive.size) or not alive[phys]:
            raise CorruptionError(f"dangling physical block id {phys}")
        bpr = self.blocks_per_row
        return frozenset((int(s) // bpr, int(s) % bpr) for s in np.nonzero(tab == phys)[0])

    def redirect(self, from_phys: int, to_phys: int) -> None:
        """Repoint every slot on from_phys to to_phys and evict from_phys (device kernel)."""
        bad = torch.zeros(1, dtype=torch.int32, device=self._table.device)
        n = self.rows * self.blocks_per_row
        if not (0 <= from_phys < n and 0 <= to_phys < n):
            raise CorruptionError(f"dangling physical block id {from_phys if not 0 <= from_phys < n else to_phys}")
        N.call(
            "kvf_table_redirect", n, N.ptr(self._table), N.ptr(self._refcount), N.ptr(self._alive),
            int(from_phys), int(to_phys), N.ptr(bad), N.stream_ptr(),
        )
        self._mutated()
        if int(bad.item()):
            raise CorruptionError(f"dangling physical block id in redirect({from_phys}, {to_phys})")

    def live_blocks(self) -> set[int]:
        return set(self.refcount)

    def audit(self) -> None:
        """Raise CorruptionError unless refcounts match the slot map (device audit kernel)."""
        from .engine import audit

        n = self.rows * self.blocks_per_row
        if not audit(self._table, self._refcount, self._alive, 1, n):
            raise CorruptionError("refcounts inconsistent with logical slot mapping")


class FusedLayer:
    """Surviving blocks of one unit: unit directions + ascending phys ids (core.py:244-258).

    ``directions`` is materialised lazily from the fused pool (device gather,
    x / |x|) as float64 numpy; ``directions_device`` keeps it on the GPU.
    """

    def __init__(self, phys_ids, loader=None, directions=None):
        # phys_ids: a sequence, or a device int32 tensor materialised on access
        self._ids = phys_ids
        self._loader = loader
        self._dirs = directions
        self._dirs_dev = None

    @property
    def phys_ids(self) -> tuple[int, ...]:
        if not isinstance(self._ids, tuple):
            src = self._ids.cpu().tolist() if isinstance(self._ids, torch.Tensor) else self._ids
            self._ids = tuple(int(i) for i in src)
        return self._ids

    @property
    def directions_device(self) -> torch.Tensor:
        if self._dirs_dev is None:
            self._dirs_dev = self._loader()
        return self._dirs_dev

    @property
    def directions(self) -> np.ndarray:
        if self._dirs is None:
            self._dirs = _to_np(self.directions_device).astype(np.float64)
        return self._dirs

    def index_of(self, phys: int) -> int:
        try:
            return self.phys_ids.index(phys)
        except ValueError:
            raise CorruptionError(f"dangling physical block id {phys}") from None


@dataclass
class FusedCache:
    """One unit's fused K/V, per-slot norms and block table (core.py:261-270).

    Device extras: the fused pools (shared by all units of the run), the
    unit index, and per-slot K/V scales s.t. K_slot = k_scale * pool[table].
    """

    keys: FusedLayer
    values: FusedLayer
    key_norms: np.ndarray
    value_norms: np.ndarray
    table: BlockTable
    block_shape: tuple[int, int, int]
    state: object = field(default=None, repr=False)
    unit: int = 0
    layer: int = 0
    head: int | None = None


class LayerView:
    """Materialised logical view (rows, blocks, t, h, d) of one layer (core.py:273-282).

    Holds numpy arrays (reference semantics); ``keys_dev``/``values_dev`` keep
    the device copies when produced by `refold`.
    """

    def __init__(self, keys, values, keys_dev: torch.Tensor | None = None,
                 values_dev: torch.Tensor | None = None):
        self._keys = keys
        self._values = values
        self.keys_dev = keys_dev
        self.values_dev = values_dev

    @property
    def keys(self) -> np.ndarray:
        if self._keys is None:
            self._keys = _to_np(self.keys_dev).astype(np.float64)
        return self._keys

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = _to_np(self.values_dev).astype(np.float64)
        return self._values

    @property
    def rows(self) -> int:
        src = self._keys if self._keys is not None else self.keys_dev
        return src.shape[0]

    @property
    def shape(self) -> tuple[int, ...]:
        src = self._keys if self._keys is not None else self.keys_dev
        return tuple(src.shape)


def refold(fused: FusedCache) -> LayerView:
    """Logical per-slot view of a fused unit (core.py:285-305), gathered on the GPU.

    Shared physical blocks are expanded once per slot and rescaled by that
    slot's own norm: K[s] = k_scale[s] * pool_k[table[s]].
    """
    fused.table.audit()
    st = fused.state
    rows, bpr = fused.key_norms.shape
    t, h, d = fused.block_shape
    g = st.geom
    dev = st.pool_k.device
    # gather the unit's vectors slot by slot: scale * x_{table[s]}
    u = fused.unit
    ids = fused.table.device_table
    out = []
    for pool, sc in ((st.pool_k, st.k_scale), (st.pool_v, st.v_scale)):
        scaled = torch.empty((ids.numel(), g.r), dtype=acc_dtype(pool.dtype), device=dev)
        N.call(
            "kvf_gather_vectors", N.ptr(pool), dtype_code(pool.dtype), *g.args(), u, N.ptr(ids),
            ids.numel(), None, N.ptr(sc[u]), N.ptr(scaled), N.stream_ptr(),
        )
        out.append(scaled.reshape(rows, bpr, t, h, d))
    return LayerView(None, None, out[0], out[1])
