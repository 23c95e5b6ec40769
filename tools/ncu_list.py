"""Summarise an ncu --metrics CSV launch list by kernel: time share and DRAM bytes."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
data = rows[hdr + 1:]
ki, ni, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
tscale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
bscale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
t, b, cnt = defaultdict(float), defaultdict(float), defaultdict(int)
for r in data:
    name = r[ki].split("(")[0].replace("void ", "")[:60]
    v = float(r[vi].replace(",", ""))
    if r[ni] == "gpu__time_duration.sum":
        t[name] += v * tscale.get(r[ui], 1.0)
        cnt[name] += 1
    elif r[ni].startswith("dram__bytes"):
        b[name] += v * bscale.get(r[ui], 1e-9)
tot = sum(t.values())
print(f"{'ms':>10} {'share':>6} {'GB':>8} {'GB/s':>8}  launches kernel")
for k, v in sorted(t.items(), key=lambda x: -x[1]):
    gbs = b[k] / (v / 1e3) if v else 0.0
    print(f"{v:10.3f} {100 * v / tot:5.1f}% {b[k]:8.2f} {gbs:8.0f}  x{cnt[k]:<4d} {k}")
print(f"{tot:10.3f} ms total")
