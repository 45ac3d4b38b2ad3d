"""Attribute stall samples of mbarrier wait loops to barrier offsets (ncu report)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, st, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = rows[2:]
tot = sum(int(r[st] or 0) for r in body if len(r) > st and (r[st] or "0").isdigit())
by = collections.Counter()
cnt = collections.Counter()
for k, r in enumerate(body):
    if "TRYWAIT" in r[si]:
        m = re.search(r"\[(R\d+)\+URZ\+(0x[0-9a-f]+)\]|\[(UR\d+)\+(0x[0-9a-f]+)\]", r[si])
        off = (m.group(2) or m.group(4)) if m else "?"
        # the sleep/poll instructions that follow belong to the same wait
        s = sum(int(body[k + d][st] or 0) for d in range(0, 4) if k + d < len(body))
        by[(k, off)] += s
        cnt[(k, off)] += int(r[ie] or 0)
print("total samples", tot)
for (k, off), s in by.most_common(20):
    print(f"  #{k:5d} bar+{off:>8s}  samples {s:7d} ({100 * s / tot:4.1f}%)  polls {cnt[(k, off)]}")
