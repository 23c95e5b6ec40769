"""Compacted fused layers: capacity, serialization and transfer.

In-place fusion keeps the standard paged layout: absorbed blocks become free
pool slots. Serving more requests per GPU, writing a fused cache to disk or
shipping it from a prefill GPU to a decode GPU wants the storage the
reference's FusedCache describes instead -- only the live blocks, in ascending
physical-id order, with `phys_ids` (core.py:246-270, fusion.py:318-327) -- so a
fused layer costs 1/CR of the unfused bytes. `compact_cache` produces it on the
device:

  kvf_alive_rank   ascending live ids + exclusive alive rank of every block
  kvf_stage_rows   live K / V rows copied densely (HBM-bound gather)
  kvf_remap_ids    slot table -> dense rows (the rank of the mapped block)

A CompactLayer decodes directly (the sharing-aware schedule is built from its
dense table; the kernel reads the compact pool), serializes to a KVFF v2 file
(`save_fused` / `load_fused`, an extension of the reference's KVFF format,
kvff.py:1-62) and moves between ranks with `send_layer` / `recv_layer`
(torch.distributed point-to-point: NCCL over NVLink on GPUs, gloo on CPU).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .attention import DecodeSchedule, _decode_sched, decode_schedule
from .engine import FusionState, Geometry, dtype_code
from .errors import ConfigError, FormatError

MAGIC = b"KVFF"
VERSION_FUSED = 2
_HEADER = struct.Struct("<4sIIIIIIII")  # magic, version, L, B, p, t, h, d, dtype code
_DT_CODE = {torch.bfloat16: 2, torch.float32: 1}
_CODE_DT = {v: k for k, v in _DT_CODE.items()}


@dataclass
class CompactLayer:
    """One fused layer stored densely: live blocks only, ascending physical id.

    keys / values: [n_live, t, h, d]; phys_ids: [n_live] the blocks' ids in
    the paged pool (FusedLayer.phys_ids); table: [B * p] dense row of every
    slot; k_scale / v_scale: [B * p] per-slot norm scales, so slot s reads
    k_scale[s] * keys[table[s]] (core.py:303-304).
    """

    layer: int
    B: int
    p_blocks: int
    keys: torch.Tensor
    values: torch.Tensor
    phys_ids: torch.Tensor
    table: torch.Tensor
    k_scale: torch.Tensor
    v_scale: torch.Tensor

    @property
    def n_live(self) -> int:
        return int(self.keys.shape[0])

    @property
    def block_shape(self) -> tuple[int, int, int]:
        return tuple(int(x) for x in self.keys.shape[1:])

    @property
    def nbytes(self) -> int:
        return sum(x.numel() * x.element_size() for x in
                   (self.keys, self.values, self.phys_ids, self.table, self.k_scale, self.v_scale))

    def pool_geometry(self) -> Geometry:
        t, h, d = self.block_shape
        return Geometry(1, self.n_live, t, h, d, 0)

    def slot_geometry(self) -> Geometry:
        t, h, d = self.block_shape
        return Geometry(1, self.B * self.p_blocks, t, h, d, 0)

    def to(self, device) -> "CompactLayer":
        return CompactLayer(self.layer, self.B, self.p_blocks,
                            *(x.to(device) for x in (self.keys, self.values, self.phys_ids,
                                                     self.table, self.k_scale, self.v_scale)))


def compact_cache(state: FusionState, B: int, p_blocks: int, layers=None) -> list[CompactLayer]:
    """Compact fused layers of a device state (folded mode, bf16 pools)."""
    g = state.geom
    if g.head_mode:
        raise ConfigError("compaction stores whole blocks: use head_mode='folded'")
    if state.pool_k.dtype != torch.bfloat16:
        raise ConfigError("compaction is implemented for bf16 pools")
    if B * p_blocks != g.NB:
        raise ConfigError(f"B*p_blocks = {B * p_blocks} does not cover the {g.NB} slots of a layer")
    dev = state.pool_k.device
    U, NB = g.units, g.NB
    live = torch.empty((U, NB), dtype=torch.int32, device=dev)
    rank = torch.empty((U, NB + 1), dtype=torch.int32, device=dev)
    count = torch.empty(U, dtype=torch.int32, device=dev)
    sp = N.stream_ptr()
    N.call("kvf_alive_rank", 0, U, NB, N.ptr(state.alive), N.ptr(live), N.ptr(rank), N.ptr(count), sp)
    n_live = count.cpu().tolist()
    out = []
    for layer in (range(g.L) if layers is None else layers):
        n = int(n_live[layer])
        keys = torch.empty((n, g.t, g.h, g.d), dtype=torch.bfloat16, device=dev)
        values = torch.empty_like(keys)
        for pool, dst in ((state.pool_k, keys), (state.pool_v, values)):
            N.call("kvf_stage_rows", N.ptr(pool), dtype_code(pool.dtype), *g.args(), layer, 1,
                   N.ptr(live), N.ptr(count), N.ptr(dst), sp)
        table = torch.empty(NB, dtype=torch.int32, device=dev)
        N.call("kvf_remap_ids", N.ptr(state.table[layer]), NB, N.ptr(rank[layer]), NB, N.ptr(table), sp)
        out.append(CompactLayer(layer, B, p_blocks, keys, values, live[layer, :n].clone(), table,
                                state.k_scale[layer].float().clone(), state.v_scale[layer].float().clone()))
    return out


def compact_decode_schedule(cl: CompactLayer, *, seq_blocks=None, item_blocks=None) -> DecodeSchedule:
    """Sharing-aware schedule of a compact layer (dense ids sort like physical ids)."""
    return decode_schedule(cl.table, cl.k_scale, cl.v_scale, cl.slot_geometry(), 0, cl.B, cl.p_blocks,
                           seq_blocks=seq_blocks, item_blocks=item_blocks)


def decode_compact(q: torch.Tensor, cl: CompactLayer, sched: DecodeSchedule, *, sm_scale=None,
                   out=None, lse=None, workspace=None, stream=None):
    """Batched decode (q [B, Hq, d]) reading the compact pool through `sched`."""
    d = cl.block_shape[2]
    sc = sm_scale if sm_scale is not None else 1.0 / float(np.sqrt(d))
    return _decode_sched(q, cl.keys, cl.values, cl.pool_geometry(), 0, cl.table, cl.k_scale,
                         cl.v_scale, sched, q.shape[1], sc, out=out, lse=lse, workspace=workspace,
                         stream=stream)


# ---------------------------------------------------------------------------
# KVFF v2: a fused cache on disk
# ---------------------------------------------------------------------------
def save_fused(path, layers: list[CompactLayer]) -> int:
    """Write compact layers as KVFF v2; returns the bytes written.

    Header (little-endian): b"KVFF", version 2, L, B, p, t, h, d, dtype code
    (1 fp32, 2 bf16); then per layer: u32 layer, u32 n_live, phys_ids u32
    [n_live], table u32 [B*p], k_scale f32 [B*p], v_scale f32 [B*p], keys and
    values [n_live, t, h, d] raw. KVFF v1 (kvff.py) holds unfused caches.
    """
    if not layers:
        raise FormatError("nothing to write")
    B, p = layers[0].B, layers[0].p_blocks
    t, h, d = layers[0].block_shape
    dt = layers[0].keys.dtype
    if dt not in _DT_CODE:
        raise FormatError(f"unsupported dtype {dt}")
    n = 0
    with open(path, "wb") as f:
        hdr = _HEADER.pack(MAGIC, VERSION_FUSED, len(layers), B, p, t, h, d, _DT_CODE[dt])
        f.write(hdr)
        n += len(hdr)
        for cl in layers:
            if (cl.B, cl.p_blocks, cl.block_shape, cl.keys.dtype) != (B, p, (t, h, d), dt):
                raise FormatError("layers of one file must share B, p, block shape and dtype")
            head = struct.pack("<II", cl.layer, cl.n_live)
            f.write(head)
            n += len(head)
            for x in (cl.phys_ids, cl.table, cl.k_scale, cl.v_scale, cl.keys, cl.values):
                b = x.contiguous().cpu().view(torch.uint8).numpy().tobytes()
                f.write(b)
                n += len(b)
    return n


def load_fused(path, device="cpu") -> list[CompactLayer]:
    """Read a KVFF v2 file written by save_fused."""
    data = Path(path).read_bytes()
    if len(data) < _HEADER.size:
        raise FormatError(f"file too short for header: {len(data)} bytes", offset=len(data))
    magic, version, L, B, p, t, h, d, code = _HEADER.unpack_from(data, 0)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {MAGIC!r}", offset=0)
    if version != VERSION_FUSED:
        raise FormatError(f"unsupported KVFF version {version} (fused caches are version 2)", offset=4)
    if code not in _CODE_DT:
        raise FormatError(f"unknown dtype code {code}", offset=32)
    dt = _CODE_DT[code]
    es = torch.empty(0, dtype=dt).element_size()
    E = t * h * d
    off = _HEADER.size
    layers = []

    def take(nbytes, what):
        nonlocal off
        if off + nbytes > len(data):
            raise FormatError(f"truncated payload reading {what}", offset=len(data))
        b = data[off:off + nbytes]
        off += nbytes
        return b

    for _ in range(L):
        layer, n_live = struct.unpack("<II", take(8, "layer header"))
        if n_live > B * p:
            raise FormatError(f"layer {layer}: {n_live} live blocks exceed {B * p} slots", offset=off - 4)

        def arr(count, dtype, what):
            raw = take(count * torch.empty(0, dtype=dtype).element_size(), what)
            return torch.frombuffer(bytearray(raw), dtype=dtype).clone() if count else torch.empty(0, dtype=dtype)

        phys = arr(n_live, torch.int32, "phys_ids")
        table = arr(B * p, torch.int32, "table")
        ks = arr(B * p, torch.float32, "k_scale")
        vs = arr(B * p, torch.float32, "v_scale")
        keys = arr(n_live * E, dt, "keys").view(n_live, t, h, d)
        values = arr(n_live * E, dt, "values").view(n_live, t, h, d)
        if n_live and (int(table.min()) < 0 or int(table.max()) >= n_live):
            raise FormatError(f"layer {layer}: table entry outside [0, {n_live})", offset=off)
        layers.append(CompactLayer(int(layer), B, p, keys, values, phys, table, ks, vs).to(device))
    if off != len(data):
        raise FormatError(f"{len(data) - off} trailing bytes after {L} layers", offset=off)
    del es
    return layers


# ---------------------------------------------------------------------------
# rank-to-rank transfer (prefill -> decode disaggregation)
# ---------------------------------------------------------------------------
def send_layer(cl: CompactLayer, dst: int, group=None) -> int:
    """Send one compact layer to rank `dst`; returns the payload bytes."""
    dev = cl.keys.device
    t, h, d = cl.block_shape
    meta = torch.tensor([cl.layer, cl.B, cl.p_blocks, t, h, d, cl.n_live, _DT_CODE[cl.keys.dtype]],
                        dtype=torch.int64, device=dev)
    dist.send(meta, dst, group=group)
    for x in (cl.phys_ids, cl.table, cl.k_scale, cl.v_scale, cl.keys, cl.values):
        dist.send(x.contiguous(), dst, group=group)
    return cl.nbytes


def recv_layer(src: int, device, group=None) -> CompactLayer:
    """Receive one compact layer sent with send_layer from rank `src`."""
    meta = torch.empty(8, dtype=torch.int64, device=device)
    dist.recv(meta, src, group=group)
    layer, B, p, t, h, d, n, code = (int(x) for x in meta.tolist())
    dt = _CODE_DT[code]
    bufs = [torch.empty(n, dtype=torch.int32, device=device),
            torch.empty(B * p, dtype=torch.int32, device=device),
            torch.empty(B * p, dtype=torch.float32, device=device),
            torch.empty(B * p, dtype=torch.float32, device=device),
            torch.empty((n, t, h, d), dtype=dt, device=device),
            torch.empty((n, t, h, d), dtype=dt, device=device)]
    for x in bufs:
        dist.recv(x, src, group=group)
    phys, table, ks, vs, keys, values = bufs
    return CompactLayer(layer, B, p, keys, values, phys, table, ks, vs)
