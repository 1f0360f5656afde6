"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals and shares."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
gi = h.index("Grid Size")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
per = []
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", "")) * scale[r[ui]]
    agg[name][0] += 1
    agg[name][1] += v
    per.append((v, name, r[gi]))
tot = sum(x[1] for x in agg.values())
print(f"total {tot:.1f} us over {sum(x[0] for x in agg.values())} launches")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:6d} {t:12.1f} us {100 * t / tot:5.1f}%  avg {t / c:9.2f} us  {k}")
if "--top" in sys.argv:
    for v, n, g in sorted(per, reverse=True)[:15]:
        print(f"  {v:9.1f} us  {n}  grid {g}")
