"""Summarise a round's GPU evidence into profiles/ (tracked):
  python tools/profile_summary.py <tag> gpurun_out/launches.csv gpurun_out/prof_attn.ncu-rep
writes profiles/<tag>_launches.txt (per-kernel launch list: count, mean device
time, share of the step), profiles/<tag>_ncu_attn.txt (key metrics of the
attention kernels from one `ncu --set full` capture) and profiles/traffic.json
(dram bytes per launch, read by bench.py's roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            h, start = r, i + 1
            break
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[start:]:
        if len(r) > vi:
            agg.setdefault(r[ki], []).append(float(r[vi].replace(",", "")))
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


KEYS = [("gpu__time_duration.sum", "time"),
        ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe % elapsed"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) % active"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("dram__bytes_read.sum", "dram read"), ("dram__bytes_write.sum", "dram write"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
        ("sm__cycles_elapsed.avg.per_second", "SM clock"),
        ("launch__registers_per_thread", "registers/thread"), ("launch__grid_size", "grid")]

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def main(tag, launches_csv, rep):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# {tag}: ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)",
             "# command: python tools/profile_step.py 2  (bench workload cfg3, 2 steps; setup kernels included)",
             f"{'kernel':80s} {'n':>3s} {'mean_us':>10s} {'share_of_skb_%':>14s}"]
    agg = launches(launches_csv)
    skb_total = sum(sum(v) for k, v in agg.items() if "skb::" in k)
    for k, v in agg.items():
        share = 100 * sum(v) / skb_total if "skb::" in k else float("nan")
        lines.append(f"{k[:80]:80s} {len(v):3d} {sum(v) / len(v) / 1e3:10.1f} {share:14.1f}")
    open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")

    h, u, rows = raw(rep)
    ki = h.index("Kernel Name")
    out = [f"# {tag}: ncu --set full --clock-control none (one launch per kernel), key metrics"]
    traffic = {}
    for r in rows:
        out.append(f"== {r[ki]}")
        for k, nm in KEYS:
            hit = [i for i, x in enumerate(h) if x == k or x.endswith("." + k)]
            if hit:
                i = hit[0]
                out.append(f"   {nm:24s} {r[i]} {u[i]}")
        rd = float(r[h.index('dram__bytes_read.sum')]) * SCALE[u[h.index('dram__bytes_read.sum')]]
        wr = float(r[h.index('dram__bytes_write.sum')]) * SCALE[u[h.index('dram__bytes_write.sum')]]
        name = r[ki].split("(")[0].split("::")[-1]
        traffic[name] = rd + wr
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_attn.txt"), "w").write("\n".join(out) + "\n")
    fwd = sum(v for k, v in traffic.items() if k.startswith("k_fwd_"))
    bwd = sum(v for k, v in traffic.items() if k.startswith("k_bwd"))
    json.dump({"attn_fwd": fwd or None, "attn_bwd": bwd or None, "per_kernel": traffic, "source": tag},
              open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print("\n".join(lines[:40]))
    print("\n".join(out))


if __name__ == "__main__":
    main(*sys.argv[1:4])
