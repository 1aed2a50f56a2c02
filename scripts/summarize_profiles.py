"""Turn gpurun_out/ ncu artefacts into committed summaries under profiles/.

usage: python scripts/summarize_profiles.py ROUND_TAG
  reads gpurun_out/launches.csv            (ncu --metrics gpu__time_duration.sum)
        gpurun_out/prof_k2_<impl>.ncu-rep  (ncu --set full, one K2 launch)
  writes profiles/<tag>_launches.txt, profiles/<tag>_k2_<impl>.txt and
         profiles/k2_traffic.json (dram bytes per K2 launch, read by bench.py)
"""

import csv
import glob
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
]


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        try:
            agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold, "
             f"serialised) of: python bench.py --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-ablation --no-kernels (k_step_bulk mixes the 15 parity-check launches at 512 sub-grids, warm-up, timed and flushed C4 steps, and e2e chunk launches)",
             f"# {'launches':>8} {'total_us':>10} {'share':>6} {'avg_us':>8}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"  {len(v):8d} {sum(v)/1e3:10.1f} {100*sum(v)/tot:5.1f}% "
                     f"{sum(v)/len(v)/1e3:8.2f}  {k}")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(tag):
    traffic = {}
    for rep in sorted(glob.glob(os.path.join(OUT, "prof_k2_*.ncu-rep"))):
        impl = os.path.basename(rep)[len("prof_k2_"):-len(".ncu-rep")]
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        hdr, units, vals = rows[0], rows[1], rows[2]
        kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        lines = [f"# ncu --set full --clock-control none, one K2 launch ({impl}): {kname[:90]}"]
        for k in KEYS:
            if k in d:
                lines.append(f"{k:80s} {d[k][1]:>14} {d[k][0]}")

        def num(k, scale_units=True):
            u, v = d.get(k, ("", "nan"))
            x = float(v.replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return x * mult
        try:
            rb, wb = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
            dur = num("gpu__time_duration.sum")
            dur_s = dur * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                           "msecond": 1e-3, "ms": 1e-3}.get(d["gpu__time_duration.sum"][0], 1e-9)
            grid = int(float(d["launch__grid_size"][1]))
            lines.append(f"# dram bytes/launch = {rb + wb:.0f}  ({(rb + wb) / dur_s / 1e9:.0f} GB/s "
                         f"over the ncu-timed launch)")
            traffic[impl] = {"dram_bytes_per_launch": rb + wb, "read": rb, "write": wb,
                             "ncu_duration_s": dur_s, "grid": grid}
        except (KeyError, ValueError):
            pass
        open(os.path.join(PROF, f"{tag}_k2_{impl}.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    # the bench's headline runs steps back to back: take the traffic of
    # back-to-back launches (ncu --cache-control none), not the cold capture
    b2b = os.path.join(OUT, "k2_b2b.txt")
    if os.path.exists(b2b) and "bulk1" in traffic:
        rd = [float(ln.split()[-1]) * 1e6 for ln in open(b2b) if "dram__bytes_read.sum" in ln]
        wr = [float(ln.split()[-1]) * 1e6 for ln in open(b2b) if "dram__bytes_write.sum" in ln]
        if rd and wr:
            traffic["bulk1"]["cold_capture_dram_bytes"] = traffic["bulk1"]["dram_bytes_per_launch"]
            traffic["bulk1"]["dram_bytes_per_launch"] = sum(rd) / len(rd) + sum(wr) / len(wr)
            traffic["bulk1"]["source"] = ("ncu --cache-control none on back-to-back launches "
                                          "(profiles/r01_k2_back_to_back.txt)")
    if traffic:
        json.dump({"tag": tag, "subgrids": 32768, "by_impl": traffic},
                  open(os.path.join(PROF, "k2_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    full(tag)
