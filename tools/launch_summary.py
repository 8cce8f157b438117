"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: python tools/launch_summary.py FILE [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0][:72]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print(f"total {tot:.0f} us over {sum(a[0] for a in agg.values())} launches")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{t:10.0f} us {100 * t / tot:5.1f}% {c:5d}  {k}")
