"""Deterministic synthetic KV caches, generated on the GPU.

Mirrors the structure of the reference generator (workload.py:144-171:
clustered block directions, K and V sharing the cluster assignment,
lognormal(0, 0.25) block norms) but replaces its Monte-Carlo noise
calibration (workload.py:89-125, minutes at r = 16,384) with the closed form
sigma_b = sqrt((1/c^2 - 1) / r), which puts each block at cosine c from its
cluster centre; c ~ U[c_lo, c_hi] per block. Test / bench infrastructure.
"""

from __future__ import annotations

import math

import torch


def _layer_blocks(gen: torch.Generator, n: int, r: int, assign: torch.Tensor, n_clusters: int,
                  c_lo: float, c_hi: float, device) -> torch.Tensor:
    bases = torch.randn((n_clusters, r), generator=gen, device=device)
    bases = bases / bases.norm(dim=1, keepdim=True)
    c = c_lo + (c_hi - c_lo) * torch.rand((n, 1), generator=gen, device=device)
    sigma = torch.sqrt((1.0 / (c * c) - 1.0) / r)
    x = bases[assign] + sigma * torch.randn((n, r), generator=gen, device=device)
    x = x / x.norm(dim=1, keepdim=True)
    norms = torch.exp(0.25 * torch.randn((n, 1), generator=gen, device=device))
    return x * norms


def synthetic_kv(L: int, B: int, p: int, t: int, h: int, d: int, *, dtype=torch.bfloat16,
                 seed: int = 0, variant: str = "bff", c_lo: float = 0.80, c_hi: float = 0.99,
                 cluster_div: int = 4, device=None, layers=None) -> tuple[torch.Tensor, torch.Tensor]:
    """K, V of shape (L, B, p, t, h, d). BFF: B*p/4 clusters per layer shared
    across requests; CFF: p/4 clusters per request (chunks of one request).

    Every layer has its own generator seeded from (seed, layer), so `layers`
    (a subset of range(L)) returns exactly those layers of the full cache,
    shape (len(layers), B, p, t, h, d) -- how bench.py hands the CPU reference
    the same bytes the GPU fused."""
    device = torch.device(device or "cuda")
    r = t * h * d
    n = B * p
    layers = list(range(L)) if layers is None else [int(x) for x in layers]
    if any(not 0 <= x < L for x in layers):
        raise ValueError(f"layers must lie in [0, {L})")
    K = torch.empty((len(layers), B, p, t, h, d), dtype=dtype, device=device)
    V = torch.empty_like(K)
    for out_i, layer in enumerate(layers):
        gen = torch.Generator(device=device)
        gen.manual_seed((seed * 1_000_003 + layer * 7919) & 0x7FFF_FFFF_FFFF)
        if variant == "bff":
            nc = max(1, n // cluster_div)
            assign = torch.randint(0, nc, (n,), generator=gen, device=device)
        else:
            per = max(1, p // cluster_div)
            nc = per * B
            assign = (torch.randint(0, per, (B, p), generator=gen, device=device)
                      + torch.arange(B, device=device)[:, None] * per).reshape(-1)
        for out in (K, V):
            blk = _layer_blocks(gen, n, r, assign, nc, c_lo, c_hi, device)
            out[out_i].copy_(blk.reshape(B, p, t, h, d).to(dtype))
    return K, V


def kv_bytes(L: int, B: int, p: int, t: int, h: int, d: int, dtype: torch.dtype) -> int:
    return 2 * L * B * p * t * h * d * torch.empty(0, dtype=dtype).element_size()


def noise_sigma(c: float, r: int) -> float:
    return math.sqrt((1.0 / (c * c) - 1.0) / r)


def synthetic_layer_into(K: torch.Tensor, V: torch.Tensor, *, seed: int = 0, c_lo: float = 0.80,
                         c_hi: float = 0.99, cluster_div: int = 4, chunk_rows: int = 8192) -> None:
    """Fill one BFF layer K, V [n, ...] in place with the synthetic_kv recipe,
    generating `chunk_rows` blocks at a time (bounded transient memory for
    caches that only just fit; the random stream differs from synthetic_kv)."""
    n = K.shape[0]
    r = K[0].numel()
    dev = K.device
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed & 0x7FFF_FFFF_FFFF)
    nc = max(1, n // cluster_div)
    assign = torch.randint(0, nc, (n,), generator=gen, device=dev)
    for out in (K, V):
        bases = torch.randn((nc, r), generator=gen, device=dev)
        bases = (bases / bases.norm(dim=1, keepdim=True)).to(torch.bfloat16)
        flat = out.view(n, r)
        for i0 in range(0, n, chunk_rows):
            i1 = min(n, i0 + chunk_rows)
            m = i1 - i0
            c = c_lo + (c_hi - c_lo) * torch.rand((m, 1), generator=gen, device=dev)
            sigma = torch.sqrt((1.0 / (c * c) - 1.0) / r)
            x = bases[assign[i0:i1]].float() + sigma * torch.randn((m, r), generator=gen, device=dev)
            x = x / x.norm(dim=1, keepdim=True)
            x = x * torch.exp(0.25 * torch.randn((m, 1), generator=gen, device=dev))
            flat[i0:i1].copy_(x.to(out.dtype))
            del x
        del bases
