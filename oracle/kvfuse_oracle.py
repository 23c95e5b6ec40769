"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference kvfuse fusion path, used by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg as the CHECKER. The product (paper_2601_03067_b200) never imports it.

Parity pinning: this module is checked against golden vectors produced by
the reference package itself (tests/golden/make_golden.py imports
/root/reference/pkg/src/kvfuse and records its outputs on the reference's own
fixtures and test cases; tests/test_oracle_golden.py asserts equality).

Each function cites the reference code it restates:
  split_norm_direction   core.py:115-119
  fuse_unit / _merge     fusion.py:205-282 (recursion 230-240, merge 242-282,
                         _unit 285-287), _fuse_layer 290-336
  BlockTable semantics   core.py:178-241 (identity 191-201, redirect 217-227)
  refold                 core.py:285-305
  paged_attention        attention.py:51-80

Decision override: when `gpu_absorber` is given, similarity
pairs with |sim - thr| <= eps are "exempt": for each right block the oracle
adopts the device's first-match decision if it is consistent with every
non-exempt pair, counts it as a flip when it differs from the float64
decision, and records a mismatch otherwise. This keeps the float64 replay in
lock-step with the device after a legitimate near-threshold flip, so tables,
refcounts and CR can be compared exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NONE = 0x7FFFFFFF


def split_norm_direction(flat: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """core.py:115-119: norms over the last axis, zero blocks keep a zero direction."""
    norms = np.sqrt(np.einsum("...i,...i->...", flat, flat))
    safe = np.where(norms > 0.0, norms, 1.0)
    return flat / safe[..., None], norms


def unit(v: np.ndarray) -> np.ndarray:
    """fusion.py:285-287."""
    n = math.sqrt(float(np.dot(v, v)))
    return v if n == 0.0 else v / n


def grouped(indices: list[int], group_size: int | None) -> list[list[int]]:
    """fusion.py:354-357."""
    if group_size is None or group_size >= len(indices):
        return [list(indices)]
    return [list(indices[i : i + group_size]) for i in range(0, len(indices), group_size)]


@dataclass
class MergeRec:
    """MergeRecord (fusion.py:93-110) + the sample moments the device reports."""

    level: int
    left_blocks: int
    right_blocks: int
    fused_count: int
    n: int
    s1: float
    s2: float
    mn: float
    mx: float
    samples: np.ndarray  # empty unless keep_samples


@dataclass
class OracleResult:
    rows: int
    bpr: int
    absorber: np.ndarray  # int32 [n], NONE if never absorbed
    table: np.ndarray  # int32 [n] slot -> phys
    refcount: np.ndarray  # int32 [n]
    alive: np.ndarray  # bool [n]
    kdir: np.ndarray  # float64 [n, r] current directions (fused for absorbers)
    vdir: np.ndarray
    key_norms: np.ndarray  # float64 [n]
    value_norms: np.ndarray
    records: list[MergeRec]
    events: list[tuple[tuple[int, int], tuple[tuple[int, int], ...]]]
    merge_calls: int
    tree_depth: int
    flips: int = 0
    mismatches: int = 0
    exempt_pairs: int = 0
    mismatch_detail: list = field(default_factory=list)

    @property
    def blocks_before(self) -> int:
        return self.rows * self.bpr

    @property
    def blocks_after(self) -> int:
        return int(self.alive.sum())

    @property
    def survivors(self) -> list[int]:
        return [int(i) for i in np.nonzero(self.alive)[0]]

    def pairs(self) -> set:
        bpr = self.bpr
        return {
            ((int(a) // bpr, int(a) % bpr), (int(j) // bpr, int(j) % bpr))
            for j, a in enumerate(self.absorber.tolist())
            if a != NONE
        }

    def samples(self) -> np.ndarray:
        arr = [m.samples for m in self.records if m.samples.size]
        return np.concatenate(arr) if arr else np.empty(0)

    def scales(self) -> tuple[np.ndarray, np.ndarray]:
        """Per-slot multipliers of the unit directions: refold uses norm[s] * dir[table[s]]."""
        return self.key_norms.copy(), self.value_norms.copy()


class _State:
    def __init__(self, kflat, vflat, rows, bpr, thr, gpu_absorber, eps, keep_samples, orig_kn, orig_vn):
        self.kdir, kn = split_norm_direction(np.asarray(kflat, dtype=np.float64))
        self.vdir, vn = split_norm_direction(np.asarray(vflat, dtype=np.float64))
        self.kn = kn if orig_kn is None else np.asarray(orig_kn, dtype=np.float64)
        self.vn = vn if orig_vn is None else np.asarray(orig_vn, dtype=np.float64)
        self.fusable = self.kn > 0.0  # fusion.py:222 (keys only)
        n = rows * bpr
        self.rows, self.bpr, self.thr = rows, bpr, thr
        self.alive = np.ones(n, dtype=bool)
        self.absorber = np.full(n, NONE, dtype=np.int64)
        # BlockTable.identity (core.py:191-201) as arrays + reverse index
        self.table = np.arange(n, dtype=np.int64)
        self.refcount = np.ones(n, dtype=np.int64)
        self.slots = {i: [i] for i in range(n)}
        self.gpu = None if gpu_absorber is None else np.asarray(gpu_absorber, dtype=np.int64)
        self.eps = eps
        self.keep_samples = keep_samples
        self.records: list[MergeRec] = []
        self.events = []
        self.merge_calls = 0
        self.flips = 0
        self.mismatches = 0
        self.exempt = 0
        self.detail = []

    def home(self, x: int) -> tuple[int, int]:
        return (x // self.bpr, x % self.bpr)

    def redirect(self, frm: int, to: int) -> None:
        """core.py:217-227."""
        moved = self.slots.pop(frm)
        for s in moved:
            self.table[s] = to
        self.slots[to].extend(moved)
        self.refcount[to] += self.refcount[frm]
        self.refcount[frm] = 0

    def fuse_rows(self, rows: list[int]) -> tuple[list[int], int]:
        """fusion.py:230-240."""
        if len(rows) == 1:
            i = rows[0]
            return [i * self.bpr + j for j in range(self.bpr)], 0
        mid = len(rows) // 2
        left, dl = self.fuse_rows(rows[:mid])
        right, dr = self.fuse_rows(rows[mid:])
        depth = max(dl, dr) + 1
        return self.merge(left, right, depth), depth

    def _decide(self, sim: np.ndarray, fl: np.ndarray, fr: np.ndarray, left: np.ndarray,
                right: np.ndarray) -> np.ndarray:
        """Per-right-block absorber index into `left` (-1 = none).

        Reference rule (fusion.py:251-265): the first left block in list order
        with sim > thr (strict) among fusable, not-yet-absorbed blocks; since
        sim is fixed for the merge this is the first qualifying row per column.
        """
        thr = self.thr
        valid = fl[:, None] & fr[None, :]
        above = (sim > thr) & valid
        first = np.where(above.any(axis=0), above.argmax(axis=0), -1)
        if self.gpu is None:
            return first
        eps = self.eps
        exempt = valid & (np.abs(sim - thr) <= eps)
        self.exempt += int(exempt.sum())
        sure = (sim > thr + eps) & valid
        pos = {int(b): k for k, b in enumerate(left.tolist())}
        out = first.copy()
        for jj, j in enumerate(right.tolist()):
            g = int(self.gpu[j])
            gi = pos.get(g, -1) if g != NONE else -1
            # GPU says absorbed by left[gi] (or by nobody when gi == -1)
            if gi >= 0:
                ok = (not sure[:gi, jj].any()) and valid[gi, jj] and (sim[gi, jj] > thr - eps)
            else:
                ok = not sure[:, jj].any()
            if ok:
                if gi != first[jj]:
                    self.flips += 1
                out[jj] = gi
            else:
                self.mismatches += 1
                if len(self.detail) < 20:
                    self.detail.append((int(j), g, int(left[first[jj]]) if first[jj] >= 0 else None))
        return out

    def merge(self, left: list[int], right: list[int], level: int) -> list[int]:
        """fusion.py:242-282."""
        self.merge_calls += 1
        la = np.asarray(left, dtype=np.int64)
        ra = np.asarray(right, dtype=np.int64)
        sim = self.kdir[la] @ self.kdir[ra].T
        fl = self.fusable[la]
        fr = self.fusable[ra]
        vals = sim[np.ix_(fl, fr)].ravel()
        samples = vals.copy() if self.keep_samples else np.empty(0)
        choice = self._decide(sim, fl, fr, la, ra)
        absorbed = choice >= 0
        fused = 0
        for li in np.unique(choice[absorbed]).tolist():  # ascending = left list order
            lid = int(la[li])
            cand = np.nonzero(choice == li)[0]
            rids = ra[cand]
            self.kdir[lid] = unit(self.kdir[lid] + self.kdir[rids].sum(axis=0))
            self.vdir[lid] = unit(self.vdir[lid] + self.vdir[rids].sum(axis=0))
            for rid in rids.tolist():
                self.redirect(int(rid), lid)
                self.alive[rid] = False
                self.absorber[rid] = lid
            fused += int(cand.size)
            self.events.append((self.home(lid), tuple(self.home(int(r)) for r in rids.tolist())))
        n_s = int(vals.size)
        self.records.append(MergeRec(
            level, int(fl.sum()), int(fr.sum()), fused, n_s, float(vals.sum()),
            float((vals * vals).sum()), float(vals.min()) if n_s else 0.0,
            float(vals.max()) if n_s else 0.0, samples))
        return left + [int(r) for j, r in enumerate(right) if not absorbed[j]]


def fuse_unit(kflat, vflat, rows: int, bpr: int, thr: float, groups: list[list[int]] | None = None,
              *, gpu_absorber=None, eps: float = 0.0, keep_samples: bool = True,
              orig_knorm=None, orig_vnorm=None) -> OracleResult:
    """Fuse one unit (a layer, or a layer x head slice): _fuse_layer, fusion.py:290-336.

    kflat / vflat: (rows*bpr, r) raw blocks; groups: independent row trees
    (default: one tree over all rows, as fast_fusion / fuse_batch without
    group_size).
    """
    if not -1.0 < thr < 1.0:
        raise ValueError(f"threshold must lie strictly inside (-1, 1), got {thr}")
    st = _State(kflat, vflat, rows, bpr, thr, gpu_absorber, eps, keep_samples, orig_knorm, orig_vnorm)
    depth = 0
    for g in groups or [list(range(rows))]:
        _, d = st.fuse_rows(list(g))
        depth = max(depth, d)
    return OracleResult(
        rows=rows, bpr=bpr, absorber=st.absorber.astype(np.int64), table=st.table.copy(),
        refcount=st.refcount.copy(), alive=st.alive.copy(), kdir=st.kdir, vdir=st.vdir,
        key_norms=st.kn, value_norms=st.vn, records=st.records, events=st.events,
        merge_calls=st.merge_calls, tree_depth=depth, flips=st.flips,
        mismatches=st.mismatches, exempt_pairs=st.exempt, mismatch_detail=st.detail,
    )


def bff_groups(B: int, group_size: int | None) -> list[list[int]]:
    """fuse_batch row groups (fusion.py:369)."""
    return grouped(list(range(B)), group_size)


def cff_groups(B: int, C: int, group_size: int | None) -> list[list[int]]:
    """fuse_chunks row groups (fusion.py:404-407)."""
    out = []
    for req in range(B):
        out.extend(grouped(list(range(req * C, (req + 1) * C)), group_size))
    return out


def cff_chunks(p: int, t: int, chunk_tokens: int) -> tuple[int, int]:
    """core.py:134-161: (C, blocks per chunk) or ValueError."""
    if chunk_tokens < 1 or chunk_tokens % t != 0 or chunk_tokens > p * t:
        raise ValueError("misaligned chunk_tokens")
    C = (p * t) // chunk_tokens
    if p % C != 0:
        raise ValueError("chunk count does not divide p")
    return C, p // C


def layer_unit(keys: np.ndarray, layer: int, head: int | None = None) -> np.ndarray:
    """(L, B, p, t, h, d) -> (B*p, r) for a layer (folded) or a layer x head."""
    x = keys[layer]
    B, p, t, h, d = x.shape
    if head is None:
        return x.reshape(B * p, t * h * d)
    return x[:, :, :, head, :].reshape(B * p, t * d)


def refold(res: OracleResult, block_shape: tuple[int, int, int]) -> tuple[np.ndarray, np.ndarray]:
    """core.py:285-305: K[s] = key_norm[s] * kdir[table[s]]."""
    t, h, d = block_shape
    k = res.key_norms[:, None] * res.kdir[res.table]
    v = res.value_norms[:, None] * res.vdir[res.table]
    shape = (res.rows, res.bpr, t, h, d)
    return k.reshape(shape), v.reshape(shape)


def softmax(z: np.ndarray) -> np.ndarray:
    """attention.py:51-55."""
    e = np.exp(z - z.max())
    return e / e.sum()


def paged_attention(q: np.ndarray, keys_view: np.ndarray, values_view: np.ndarray, row: int,
                    head: int) -> tuple[np.ndarray, np.ndarray]:
    """attention.py:58-80 over a (rows, p, t, h, d) view."""
    _, p, t, h, d = keys_view.shape
    K = keys_view[row, :, :, head, :].reshape(p * t, d)
    V = values_view[row, :, :, head, :].reshape(p * t, d)
    s = softmax(K @ q / np.sqrt(d))
    return s @ V, s
