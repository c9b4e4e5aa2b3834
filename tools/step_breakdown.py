#!/usr/bin/env python3
"""Per-kernel-family device time and DRAM traffic of one bench step, from an ncu launch
list (gpu__time_duration.sum + dram bytes), taken with

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --cache-control none --clock-control none --csv --log-file L.csv \\
        python bench.py --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline \\
        --no-kprof --no-parity --no-producer

The process launches (warmup + steps) identical steps; the last 1/(warmup+steps) of our
launches is the measured step. Launches are classified by kernel name into the families
bench.py times (FAMILY_BPE): the on-chip single-launch passes (k_onchip, forward /
backward by its BWD template flag), statistics and backward reductions (k_reduce_*,
k_fold_rows over StatsOp / BwdOp) and the elementwise passes with their finalize kernels
(k_ew_affine, k_finalize_fwd -> fwd_normalize; k_ew_dx, k_finalize_bwd -> bwd_dx).

    python tools/step_breakdown.py L.csv [--passes 4]            # family table
    python tools/step_breakdown.py L.csv --traffic out.json [--passes 4]
"""
import argparse
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import FAMILY_BPE  # noqa: E402

OURS = ("k_onchip", "k_reduce", "k_fold_rows", "k_ew_", "k_finalize")


def family(name):
    if "k_onchip" in name:
        # k_onchip<T, VE, BWD, RELU>: the third template argument
        args = re.search(r"k_onchip<([^>]*)>", name).group(1).split(",")
        return "bwd_onchip" if args[2].strip() in ("1", "(bool)1", "true") else "fwd_onchip"
    if "k_reduce" in name or "k_fold_rows" in name:
        return "bwd_reduce" if "BwdOp" in name or "BwdRows" in name else "fwd_stats"
    if "k_ew_affine" in name or "k_finalize_fwd" in name or "k_finalize_sums" in name:
        return "fwd_normalize"
    if "k_ew_dx" in name or "k_finalize_bwd" in name:
        return "bwd_dx"
    return None


def load_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    k = {}
    for r in rows[1:]:
        d = k.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return [k[i] for i in sorted(k) if any(t in k[i]["name"] for t in OURS)]


def step_families(path, passes):
    ours = load_launches(path)
    per = len(ours) // passes
    step = ours[-per:]
    fam = {}
    for kk in step:
        f = family(kk["name"])
        if f is None:
            continue
        fam.setdefault(f, []).append(kk)
    return fam, per


def summarise(fam):
    tot_t = sum(kk["gpu__time_duration.sum"] for v in fam.values() for kk in v)
    res = {}
    for name, v in fam.items():
        dram = sum(kk.get("dram__bytes_read.sum", 0) + kk.get("dram__bytes_write.sum", 0)
                   for kk in v)
        t = sum(kk["gpu__time_duration.sum"] for kk in v)
        res[name] = {"launches": len(v), "dram_bytes_per_launch": dram / len(v),
                     "ncu_time_us_per_step": t / 1e3, "ncu_share": t / tot_t,
                     "dram_gbs": dram / t if t else None, "bytes_per_elem": FAMILY_BPE[name]}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic", default=None, help="write the per-family JSON here")
    ap.add_argument("--passes", type=int, default=4, help="warmup + timed steps in the run")
    a = ap.parse_args()
    fam, per = step_families(a.csv, a.passes)
    res = summarise(fam)
    if a.traffic:
        doc = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                         "dram__bytes_write.sum --cache-control none --clock-control none on "
                         "`python bench.py --steps 1 --warmup 3 --no-graph --no-e2e "
                         "--no-cpu-baseline --no-kprof --no-parity --no-producer` (one eager "
                         "step; launches classified by kernel name). Per-launch dram bytes "
                         "include write-backs of lines the previous kernel left dirty in L2.",
               "launch_list": os.path.basename(a.csv), "launches_per_step": per,
               "families": res}
        json.dump(doc, open(a.traffic, "w"), indent=1)
    print(f"{'family':>14} {'launches':>8} {'ncu us':>9} {'share':>6} {'dram MB/launch':>14}"
          f" {'dram GB/s':>9}")
    for name, v in sorted(res.items(), key=lambda kv: -kv[1]["ncu_time_us_per_step"]):
        print(f"{name:>14} {v['launches']:8d} {v['ncu_time_us_per_step']:9.1f} "
              f"{v['ncu_share']:6.3f} {v['dram_bytes_per_launch'] / 1e6:14.2f} "
              f"{(v['dram_gbs'] or 0):9.0f}")
    print(f"launches per step: {per}")


if __name__ == "__main__":
    main()
