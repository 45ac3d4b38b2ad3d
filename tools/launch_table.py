"""Per-kernel mean device time from an ncu --metrics gpu__time_duration.sum csv."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, start = r, i + 1
        break
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[start:]:
    if len(r) > vi:
        agg.setdefault(r[ki], []).append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print(f"{k[:70]:70s} n={len(v):3d} mean_us={sum(v) / len(v) / 1e3:9.1f}")
