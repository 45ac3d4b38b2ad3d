"""Top stalled SASS instructions of an ncu report (with the stall reason columns)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, st, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reason_cols = [i for i, x in enumerate(h) if x.startswith("stall_") or "Stall" in x and "Samples" not in x]
data = []
for idx, r in enumerate(rows[2:]):
    try:
        data.append((int(r[st] or 0), int(r[ie] or 0), idx, r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total stall samples", tot)
for s, e, idx, src in sorted(data, reverse=True)[:n]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  #{idx:5d} inst={e:10d}  {src[:90]}")
