"""Mean duration per kernel name of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
d = defaultdict(list)
for r in rows[1:]:
    d[r[iN].split("(")[0][:70]].append(float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0))
for k, v in d.items():
    print(f"{k:70s} n={len(v):4d} mean={sum(v) / len(v):9.2f} us")
