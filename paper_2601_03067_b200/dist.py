"""Multi-GPU plumbing for the fusion path.

Fusion is independent per layer (fusion.py:367-374) and, in per-head mode,
per (layer, KV head), so ranks shard units and never exchange KV data. The
only collectives are the ones the north star names: gathering compression
statistics (per-unit block counts) and, optionally, the remapped block tables.
One process per GPU, torch.distributed over NCCL (gloo for CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def shard_units(n_units: int, world: int, rank: int) -> range:
    """Contiguous, balanced unit range of `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_units, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass
class CompressionStats:
    blocks_before: int
    blocks_after: int
    per_rank_after: list[int]

    @property
    def compression_ratio(self) -> float:
        return self.blocks_before / self.blocks_after


def gather_compression(blocks_before: torch.Tensor, blocks_after: torch.Tensor,
                       group=None) -> CompressionStats:
    """All-gather per-unit (before, after) block counts; aggregate CR = sum / sum
    (FusionReport.aggregate, fusion.py:158-171). Tensors are int64 [units_local]
    on the backend's device (CUDA for NCCL, CPU for gloo)."""
    world = dist.get_world_size(group)
    local = torch.stack([blocks_before.sum(), blocks_after.sum()]).to(torch.int64)
    out = torch.empty(world * 2, dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    per = out.view(world, 2).cpu().tolist()
    return CompressionStats(sum(p[0] for p in per), sum(p[1] for p in per), [p[1] for p in per])


def gather_tables(table: torch.Tensor, dst: int = 0, group=None) -> list[torch.Tensor] | None:
    """Gather every rank's remapped int32 tables [units_local, NB] to `dst`
    (units may differ by one between ranks)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = torch.tensor([table.shape[0]], dtype=torch.int64, device=table.device)
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    rows = max(int(s.item()) for s in sizes)
    padded = torch.zeros((rows, table.shape[1]), dtype=table.dtype, device=table.device)
    padded[: table.shape[0]] = table
    bufs = [torch.empty_like(padded) for _ in range(world)] if rank == dst else None
    dist.gather(padded, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return [b[: int(s.item())] for b, s in zip(bufs, sizes)]


def _coll_device(group=None) -> torch.device:
    """Tensors for collectives: CUDA for NCCL, host for gloo."""
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


@dataclass
class ShardedFusion:
    """One rank's share of a layer-sharded fusion run (fuse_batch_sharded)."""

    layers: range  # this rank's layers of the cache
    outcomes: list  # FusionOutcome per local unit (layer, or layer x kv head)
    stats: CompressionStats  # all ranks: aggregate blocks before / after, per-rank after
    tables: list[torch.Tensor] | None  # on `dst`: every rank's int32 tables [units_r, NB]


def fuse_batch_sharded(cache, cfg, *, group=None, gather: bool = True, dst: int = 0,
                       **kwargs) -> ShardedFusion:
    """BFF (or CFF with cfg.variant == "cff" and chunk_tokens=) over the layers of this
    rank's shard (fusion.py:367-374: layers are independent), then the path's only
    collectives: an all-gather of the per-unit block counts and, with `gather`, a
    gather of the remapped int32 tables to `dst`. Every rank holds the whole cache
    description; only its layers are read (device caches: views; host-resident
    caches: only these layers are streamed). Returns this rank's ShardedFusion."""
    from .fusion import fuse_batch, fuse_chunks

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = shard_units(cache.dims.L, world, rank)
    chunk_tokens = kwargs.pop("chunk_tokens", None)
    if cfg.variant == "cff":
        outs = fuse_chunks(cache, cfg, chunk_tokens, layers=mine, **kwargs)
    else:
        outs = fuse_batch(cache, cfg, layers=mine, **kwargs)
    cd = _coll_device(group)
    before = torch.tensor([o.report.blocks_before for o in outs], dtype=torch.int64, device=cd)
    after = torch.tensor([o.report.blocks_after for o in outs], dtype=torch.int64, device=cd)
    stats = gather_compression(before, after, group=group)
    tables = None
    if gather:
        local = torch.stack([o.fused.table.device_table for o in outs]).to(cd)
        tables = gather_tables(local, dst=dst, group=group)
    return ShardedFusion(mine, outs, stats, tables)
