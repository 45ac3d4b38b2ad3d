"""Stall-reason totals of one kernel in an ncu report (source page), and the
top instructions per reason: python tools/ncu_stalls.py rep.ncu-rep kernel_regex [n]."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 6
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r]
h = rows[hi[0]]
data = rows[hi[0] + 1:(hi[1] if len(hi) > 1 else len(rows))]
si, ie = h.index("Source"), h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: 0 for c in cols}
per = {c: [] for c in cols}
for k, r in enumerate(data):
    for c in cols:
        try:
            v = int(r[h.index(c)] or 0)
        except (ValueError, IndexError):
            continue
        tot[c] += v
        per[c].append((v, k, r[si].strip()[:70]))
T = sum(tot.values())
print("samples", T)
for c, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v == 0:
        continue
    print(f"{c:24s} {v:8d} {100 * v / T:5.1f}%")
    for vv, k, src in sorted(per[c], reverse=True)[:n]:
        print(f"      {vv:7d} #{k:5d} {src}")
