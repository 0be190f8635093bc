"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    k = r[ki].split("(")[0][:80]
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:6d} {v[1] / 1e3:10.1f}us {100 * v[1] / tot:5.1f}% avg {v[1] / v[0] / 1e3:8.2f}us {k}")
