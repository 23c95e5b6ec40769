"""Paged decode attention over fused caches -- drop-in for kvfuse.attention.

`paged_attention` keeps the reference signature (attention.py:58-80): one
query against one KV head of one request, exact softmax, returning the output
and the probability vector. It runs on the GPU through K6
(`kvf_paged_decode`), which reads K/V through the block table with per-slot
scales, so it accepts either a refolded `LayerView` or a `FusedCache`
directly. `paged_decode` is the batched serving form: all requests x all
query heads (GQA) of one layer in one launch pair.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .core import FusedCache, LayerView, default_device
from .engine import Geometry, FusionState, acc_dtype, dtype_code
from .errors import DomainError, InvalidCacheError


@dataclass(frozen=True)
class AttentionQuery:
    """A single-head query against one layer (attention.py:20-32)."""

    q: np.ndarray
    head: int = 0
    layer: int = 0

    def __post_init__(self):
        q = np.asarray(self.q, dtype=np.float64)
        if q.ndim != 1 or not np.isfinite(q).all():
            raise InvalidCacheError("query must be a finite 1-D vector")
        object.__setattr__(self, "q", q)


@dataclass(frozen=True)
class SoftmaxDistribution:
    """Probability vector over attended tokens (attention.py:35-48)."""

    probs: np.ndarray

    def __post_init__(self):
        probs = np.asarray(self.probs, dtype=np.float64)
        if probs.ndim != 1 or (probs < 0).any() or abs(probs.sum() - 1.0) > 1e-9:
            raise InvalidCacheError("softmax output must be a probability vector")
        object.__setattr__(self, "probs", probs)

    def __len__(self) -> int:
        return len(self.probs)


def softmax(z: np.ndarray) -> np.ndarray:
    """Max-subtracted softmax of host logits (attention.py:51-55)."""
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - z.max())
    return e / e.sum()


def attention_drift(s: SoftmaxDistribution, s_prime: SoftmaxDistribution) -> float:
    """L1 distance between two attention distributions (attention.py:83-87)."""
    if len(s) != len(s_prime):
        raise DomainError(f"distribution lengths differ: {len(s)} vs {len(s_prime)}")
    return float(np.abs(s_prime.probs - s.probs).sum())


def _decode(q: torch.Tensor, pool_k, pool_v, geom: Geometry, layer: int, table, k_scale,
            v_scale, B: int, p_blocks: int, Hq: int, sm_scale: float, *, seq_blocks=None,
            want_probs: bool = False, out=None, lse=None, workspace=None, stream=None):
    dt = dtype_code(pool_k.dtype)
    acc = acc_dtype(pool_k.dtype)
    dev = pool_k.device
    if out is None:
        out = torch.empty((B, Hq, geom.d), dtype=acc, device=dev)
    if lse is None:
        lse = torch.empty((B, Hq), dtype=acc, device=dev)
    probs = torch.empty((B, Hq, p_blocks * geom.t), dtype=acc, device=dev) if want_probs else None
    ws_bytes = N.lib().kvf_decode_workspace_size(dt, B, Hq, geom.d, p_blocks, geom.t)
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    N.call(
        "kvf_paged_decode", N.ptr(q), dtype_code(q.dtype), N.ptr(pool_k), N.ptr(pool_v), dt,
        *geom.args(), layer, N.ptr(table), N.ptr(k_scale), N.ptr(v_scale), B, p_blocks,
        N.ptr(seq_blocks), Hq, float(sm_scale), N.ptr(out), N.ptr(lse), N.ptr(probs),
        N.ptr(workspace), workspace.numel(), N.stream_ptr(stream),
    )
    return out, lse, probs


def paged_decode(q: torch.Tensor, state: FusionState, layer: int, B: int, p_blocks: int, *,
                 sm_scale: float | None = None, seq_blocks: torch.Tensor | None = None,
                 out=None, lse=None, workspace=None, stream=None):
    """Batched decode over a fused device state: q [B, Hq, d] -> out [B, Hq, d].

    Slot (b, j) = b * p_blocks + j of `layer`; Hq must be a multiple of the
    KV head count (GQA group = Hq / h).
    """
    g = state.geom
    Hq = q.shape[1]
    sc = sm_scale if sm_scale is not None else 1.0 / float(np.sqrt(g.d))
    o, l, _ = _decode(q, state.pool_k, state.pool_v, g, layer, state.table, state.k_scale,
                      state.v_scale, B, p_blocks, Hq, sc, seq_blocks=seq_blocks, out=out,
                      lse=lse, workspace=workspace, stream=stream)
    return o, l


def paged_attention(query: AttentionQuery, view, row: int = 0):
    """Exact softmax attention over all logical tokens of one request (attention.py:58-80).

    ``view`` is a refolded LayerView (rows, blocks, t, h, d) or a FusedCache
    (read through its table with per-slot norm scales, no refold needed).
    """
    if isinstance(view, FusedCache):
        return _attention_fused(query, view, row)
    if not isinstance(view, LayerView):
        raise InvalidCacheError("view must be a LayerView or a FusedCache")
    keys_dev, values_dev = view.keys_dev, view.values_dev
    dev = default_device()
    if keys_dev is None:
        keys_dev = torch.from_numpy(np.ascontiguousarray(view.keys, dtype=np.float64)).to(dev)
        values_dev = torch.from_numpy(np.ascontiguousarray(view.values, dtype=np.float64)).to(dev)
    if keys_dev.numel() == 0:
        raise InvalidCacheError("empty cache view")
    rows, p, t, h, d = keys_dev.shape
    if not 0 <= row < rows:
        raise InvalidCacheError(f"row {row} out of range [0, {rows})")
    if not 0 <= query.head < h:
        raise InvalidCacheError(f"head {query.head} out of range [0, {h})")
    if query.q.shape != (d,):
        raise InvalidCacheError(f"query length {query.q.shape} does not match head size {d}")
    geom = Geometry(1, rows * p, t, h, d, 0)
    acc = acc_dtype(keys_dev.dtype)
    table = torch.zeros(rows * p, dtype=torch.int32, device=keys_dev.device)
    table[:p] = torch.arange(row * p, (row + 1) * p, dtype=torch.int32, device=keys_dev.device)
    ones = torch.ones(rows * p, dtype=acc, device=keys_dev.device)
    return _single(query, keys_dev.contiguous(), values_dev.contiguous(), geom, 0, table, ones,
                   ones, p, query.head, h)


def _attention_fused(query: AttentionQuery, fused: FusedCache, row: int):
    st: FusionState = fused.state
    g = st.geom
    rows, bpr = fused.key_norms.shape
    t, hb, d = fused.block_shape
    if not 0 <= row < rows:
        raise InvalidCacheError(f"row {row} out of range [0, {rows})")
    if not 0 <= query.head < hb:
        raise InvalidCacheError(f"head {query.head} out of range [0, {hb})")
    if query.q.shape != (d,):
        raise InvalidCacheError(f"query length {query.q.shape} does not match head size {d}")
    # one logical request = `row` of this unit; present it as request 0
    u = fused.unit
    tab = st.table[u]
    table = torch.zeros_like(st.table)
    ks = torch.zeros_like(st.k_scale)
    vs = torch.zeros_like(st.v_scale)
    sl = slice(row * bpr, (row + 1) * bpr)
    table[u, :bpr] = tab[sl]
    ks[u, :bpr] = st.k_scale[u, sl]
    vs[u, :bpr] = st.v_scale[u, sl]
    kv_head = fused.head if g.head_mode else query.head
    return _single(query, st.pool_k, st.pool_v, g, fused.layer, table, ks, vs, bpr, kv_head, g.h)


def _single(query, pool_k, pool_v, geom, layer, table, ks, vs, p_blocks, kv_head, h):
    acc = acc_dtype(pool_k.dtype)
    dev = pool_k.device
    q = torch.zeros((1, h, geom.d), dtype=acc, device=dev)
    q[0, kv_head] = torch.from_numpy(query.q).to(dev, acc)
    out, _, probs = _decode(q, pool_k, pool_v, geom, layer, table, ks, vs, 1, p_blocks, h,
                            1.0 / float(np.sqrt(geom.d)), want_probs=True)
    o = out[0, kv_head].double().cpu().numpy()
    pr = probs[0, kv_head].double().cpu().numpy()
    pr = pr / pr.sum()
    return o, SoftmaxDistribution(pr)
