#!/usr/bin/env python3
"""Key metrics per kernel from ncu --set full reports (first launch of each kernel name):
    python tools/ncu_summary.py rep1.ncu-rep [rep2.ncu-rep ...] > profiles/rNN_ncu_full_summary.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__cluster_dim_x",
    "launch__occupancy_limit_registers",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    seen = set()
    print(f"# {rep}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if name in seen:
            continue
        seen.add(name)
        print(f"## {name[:150]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:74s} {r[i]:>14} {units[i]}")
