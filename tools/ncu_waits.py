"""Stall samples per mbarrier wait site of an ncu report (sm_100 SASS source page).
usage: python tools/ncu_waits.py report.ncu-rep kernel_regex bar_base_offset name,name,..."""
import csv
import io
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
base = int(sys.argv[3]) if len(sys.argv) > 3 else None
names = sys.argv[4].split(",") if len(sys.argv) > 4 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
si, st = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
tot = sum(int(r[st] or 0) for r in data)
acc = {}
i = 0
while i < len(data):
    s = data[i][si]
    if "SYNCS.PHASECHK" in s and "TRYWAIT" in s:
        m = re.search(r"\+(0x[0-9a-f]+)\]", s)
        off = int(m.group(1), 16) if m else -1
        samples = sum(int(data[j][st] or 0) for j in range(i, min(i + 4, len(data))))
        tag = hex(off)
        if base is not None and off >= base and (off - base) % 8 == 0 and (off - base) // 8 < len(names):
            tag = names[(off - base) // 8]
        acc.setdefault(tag, [0, 0])
        acc[tag][0] += samples
        acc[tag][1] += int(data[i][ie] or 0)
    i += 1
print("total samples", tot)
for k, (s, n) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"{k:12s} {s:8d} {100 * s / tot:5.1f}%  waits={n}")
