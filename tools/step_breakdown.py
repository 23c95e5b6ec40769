"""Warm per-launch breakdown of one cfg2-shaped fusion step: CUDA events around every
C-ABI call of an eager FusionEngine.run (same stream, so the intervals tile the step).

usage: python tools/step_breakdown.py [L] [B] [p] [exact:on|off] [compact_from|auto|none] [staged|gathered]
"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_03067_b200 import _native as N  # noqa: E402
from paper_2601_03067_b200.engine import FusionEngine, Geometry  # noqa: E402
from paper_2601_03067_b200.schedule import bff_plan  # noqa: E402
from paper_2601_03067_b200.workload import synthetic_kv  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
p = int(sys.argv[3]) if len(sys.argv) > 3 else 256
exact = (sys.argv[4] != "off") if len(sys.argv) > 4 else None
cf = sys.argv[5] if len(sys.argv) > 5 else "auto"
cf = None if cf == "none" else ("auto" if cf == "auto" else int(cf))
cmode = sys.argv[6] if len(sys.argv) > 6 else "auto"
t, h, d = 16, 8, 128
variant = os.environ.get("VARIANT", "bff")  # cff: chunks of 2048 tokens (cfg3 = 32 1 1024)
DT = torch.float32 if os.environ.get("DTYPE") == "f32" else torch.bfloat16  # cfg1: DTYPE=f32 4 8 64
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=DT, seed=1000, variant=variant)
Kt, Vt = Kt.reshape(-1), Vt.reshape(-1)
geom = Geometry(L, B * p, t, h, d, int(os.environ.get("HEAD_MODE", "0")))
if variant == "cff":
    from paper_2601_03067_b200.core import cff_layout
    from paper_2601_03067_b200.schedule import cff_plan

    C, bpc = cff_layout(p, t, 2048)
    plan = cff_plan(B, C, bpc, None)
else:
    plan = bff_plan(B, p, None)
eng = FusionEngine(geom, plan, DT, Kt.device, N.PATH_TC, exact=exact, compact_from=cf,
                   compact_mode=cmode)
k, v = Kt.clone(), Vt.clone()

_orig = N.call
rec = []


def timed(name, *a, **kw):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _orig(name, *a, **kw)
    e1.record()
    rec.append((name, e0, e1))


for it in range(3):
    k.copy_(Kt)
    v.copy_(Vt)
    rec.clear()
    N.call = timed if it == 2 else _orig
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    st = eng.run(k, v, 0.8)
    s1.record()
    torch.cuda.synchronize()
N.call = _orig
tot = collections.defaultdict(float)
cnt = collections.Counter()
seq = []
for name, a, b in rec:
    ms = a.elapsed_time(b)
    tot[name] += ms
    cnt[name] += 1
    seq.append((name, ms))
step = s0.elapsed_time(s1)
print(f"L={L} B={B} p={p} exact={eng.exact} compact_from={eng.compact_from} mode={eng.compact_mode} "
      f"CR {(U0 := geom.units * geom.NB) / max(int(st.live_count.sum()), 1):.6f} step {step:.2f} ms "
      f"(sum of calls {sum(tot.values()):.2f})")
for name in sorted(tot, key=lambda n: -tot[n]):
    print(f"  {tot[name]:8.2f} ms  {100 * tot[name] / step:5.1f}%  x{cnt[name]:<3d} {name}")
print("sequence:")
for name, ms in seq:
    if ms > 0.05:
        print(f"  {ms:8.3f}  {name}")

# algorithmic merge bytes per level: items = (absorber, K|V); reads = absorber + members,
# one write per item; exact mode: key vectors with a shadow row are read as fp32 rows and
# every key absorber also writes its fp32 row
U, NB = geom.units, geom.NB
ab = st.absorber.long()
vb = geom.r * Kt.element_size()
seen_abs = torch.zeros((U, NB), dtype=torch.bool, device=ab.device)
merge_ms = [ms for name, ms in seq if name == "kvf_merge_groups"]
blk = torch.arange(NB, device=ab.device)
for li, lv in enumerate(plan.levels):
    m = torch.from_numpy(lv.row_merge).to(ab.device).long()[blk // plan.bpr]
    mg = torch.from_numpy(lv.merges).to(ab.device).long()
    ok = m >= 0
    lb, mid = mg[m.clamp(min=0), 0], mg[m.clamp(min=0), 1]
    member = ok & (blk >= mid) & (ab >= lb) & (ab < mid) & (ab != 0x7FFFFFFF)
    member = member.expand(U, NB) if member.dim() == 1 else member
    n_mem = int(member.sum())
    absr = torch.zeros((U, NB), dtype=torch.bool, device=ab.device)
    uu = torch.arange(U, device=ab.device)[:, None].expand(U, NB)
    absr[uu[member], ab[member]] = True
    n_abs = int(absr.sum())
    base = 2 * (n_abs + n_mem) * vb + 2 * n_abs * vb  # K and V: reads + writes
    extra = 0
    if eng.exact:
        sh_mem = int((member & seen_abs).sum())
        sh_abs = int((absr & seen_abs).sum())
        last = li == len(plan.levels) - 1  # the last level writes no shadow rows
        extra = (sh_mem + sh_abs) * vb + (0 if last else n_abs * 2 * vb)  # fp32 reads (2x) + row writes
    seen_abs |= absr
    gb = (base + extra) / 1e9
    ms = merge_ms[li] if li < len(merge_ms) else float("nan")
    print(f"level {li + 1}: absorbers {n_abs} members {n_mem} merge bytes {gb:.2f} GB "
          f"({ms:.3f} ms -> {gb / ms:.2f} TB/s algorithmic)")

# similarity work per level: algorithmic FLOPs (alive fusable pairs) vs executed FLOPs
# (active 256 x 256 tiles: full rectangles over pool rows, or over alive rows when compacted)
sim_ms = collections.defaultdict(float)
lvl_of = []
li = 0
for name, ms in seq:
    if name == "kvf_similarity_select":
        sim_ms[li] += ms
    if name == "kvf_merge_groups":
        li += 1
alive_hist = []  # alive flags before each level, reconstructed from the absorber record
alive = torch.ones((U, NB), dtype=torch.bool, device=ab.device)
for li, lv in enumerate(plan.levels):
    s_ = st.level_stats[li].double()
    alg = float((2 * s_[..., 0] * s_[..., 1]).sum()) * geom.r
    mg = torch.from_numpy(lv.merges).to(ab.device).long()
    compact = eng.compact_from is not None and lv.height >= eng.compact_from
    ex_tiles = 0
    cum = torch.cat([torch.zeros((U, 1), dtype=torch.long, device=ab.device), alive.long().cumsum(1)], 1)
    for lb_, mid_, re_ in mg.tolist():
        if compact:
            nl = (cum[:, mid_] - cum[:, lb_]).clamp(min=0)
            nr = (cum[:, re_] - cum[:, mid_]).clamp(min=0)
        else:
            nl = torch.full((U,), mid_ - lb_, device=ab.device)
            nr = torch.full((U,), re_ - mid_, device=ab.device)
        ex_tiles += int(((nl + 255) // 256 * ((nr + 255) // 256)).sum())
    exe = ex_tiles * 2.0 * 256 * 256 * geom.r
    ms = sim_ms[li]
    print(f"level {li + 1}: sim {ms:.3f} ms  algorithmic {alg / 1e12:.2f} TFLOP ({alg / ms / 1e9:.0f} TF/s)  "
          f"executed {exe / 1e12:.2f} TFLOP ({exe / ms / 1e9:.0f} TF/s, {alg / exe:.2f} useful)")
    # blocks absorbed at this level die before the next
    m = torch.from_numpy(lv.row_merge).to(ab.device).long()[blk // plan.bpr]
    lb, mid = mg[m.clamp(min=0), 0], mg[m.clamp(min=0), 1]
    member = (m >= 0) & (blk >= mid) & (ab >= lb) & (ab < mid) & (ab != 0x7FFFFFFF)
    alive &= ~member
