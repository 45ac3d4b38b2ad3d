"""Summarise an ncu report: duration, pipes, stall reasons, SASS opcode histogram."""
import collections
import csv
import io
import re
import subprocess
import sys


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, top=18):
    raw = page(rep, "raw")
    h, v = raw[0], raw[2]
    get = {n: v[i] for i, n in enumerate(h)}
    keys = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size"]
    for k in keys:
        for n in get:
            if n.endswith(k):
                print(f"{n:90s} {get[n]}")
                break
    st = sorted(((float(get[n]), n) for n in get if "pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued")
                 and get[n].replace('.', '', 1).isdigit()), reverse=True)[:8]
    for val, n in st:
        print(f"  stall {val:10.0f} {n.split('stalled_')[-1]}")
    src = page(rep, "source")
    hh = src[1]
    ia, so, sa = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
    ops, stl, tot = collections.Counter(), collections.Counter(), 0
    for r in src[2:]:
        try:
            n, s = int(r[ia]), int(r[sa])
        except (ValueError, IndexError):
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[so])
        op = m.group(2) if m else "?"
        ops[op] += n
        stl[op] += s
        tot += n
    print(f"  warp instructions {tot}")
    for op, n in ops.most_common(top):
        print(f"  {op:10s} {n:12d} {100 * n / tot:5.1f}%  stall-samples {stl[op]}")


if __name__ == "__main__":
    main(sys.argv[1])
