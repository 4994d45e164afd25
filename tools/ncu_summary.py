#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>            -> per-kernel launch table
  python tools/ncu_summary.py report <file.ncu-rep> [label]      -> key counters per kernel
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_us"),
    ("dram__bytes_read.sum", "dram_read_B"),
    ("dram__bytes_write.sum", "dram_write_B"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("smsp__inst_executed_pipe_fma.sum", "inst_pipe_fma"),
    ("smsp__inst_executed.sum", "inst_executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("smsp__sass_average_branch_targets_threads_uniform.pct", "branch_uniform_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def launches(path: str):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    agg = collections.defaultdict(list)
    for r in rows:
        agg[(r[ki].split("(")[0][:70], r[gi])].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'launches':>8} {'avg_us':>9} {'share':>6}  kernel [grid]")
    for (k, gsz), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {100 * sum(v) / tot:5.1f}%  {k} {gsz}")


def report(path: str, label: str = ""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    unit_of = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    name_i = hdr.index("Kernel Name")
    print(f"# ncu --set full summary {label}".rstrip())
    for r in rows[2:]:
        vals = dict(zip(hdr, r))
        print(f"\n## {vals[hdr[name_i]][:110]}")
        for k, short in KEYS:
            if k in vals:
                v = vals[k]
                u = unit_of.get(k, "")
                if u in scale and v:   # bytes in bytes, durations in us
                    v = f"{float(v.replace(',', '')) * scale[u]:.6g}"
                print(f"  {short:22s} {v}")
        stalls = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                          float(v.replace(",", "") or 0)) for h, v in vals.items()
                         if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")),
                        key=lambda t: -t[1])
        print("  stalls/issue          " + ", ".join(f"{n}={v:.2f}" for n, v in stalls[:6]))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
