"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]; data = rows[hdr + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg, cnt = defaultdict(float), defaultdict(int)
for r in data:
    name = r[ki].split("(")[0].replace("void ", "")[:70]
    agg[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v:10.3f} ms {100 * v / tot:5.1f}%  x{cnt[k]:<4d} {k}")
print(f"{tot:10.3f} ms total")
