#!/usr/bin/env python3
"""Aggregate an ncu launch list (gpu__time_duration.sum per kernel) of one bench step
into per-layer / per-kernel-type times. Usage: step_breakdown.py launches.csv [n_skip]"""
import csv
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import resnet50_bn_shapes, numel  # noqa: E402

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
ks = [(r[ki], float(r[vi])) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
ours = [(n, t) for n, t in ks if "k_" in n and ("reduce" in n or "affine" in n or "dx" in n or "fused" in n)]
shapes = resnet50_bn_shapes(32)
per_step = 4 * len(shapes)
step = ours[-per_step:]
def kind(n):
    if "StatsOp" in n: return "stats"
    if "BwdOp" in n: return "bwd_reduce"
    if "affine" in n: return "normalize"
    if "dx" in n: return "bwd_dx"
    return n[:30]
fwd = step[:2 * len(shapes)]
bwd = step[2 * len(shapes):]
tot = {}
print(f"{'layer':>5} {'shape':>22} {'MB':>7} {'stats':>7} {'norm':>7} {'bred':>7} {'dx':>7} {'sum us':>8} {'alg GB/s':>9}")
grand = 0.0
for li, s in enumerate(shapes):
    st, nm = fwd[2 * li], fwd[2 * li + 1]
    bi = len(shapes) - 1 - li
    br, dx = bwd[2 * bi], bwd[2 * bi + 1]
    ts = [st[1] / 1e3, nm[1] / 1e3, br[1] / 1e3, dx[1] / 1e3]
    for k, t in zip(("stats", "normalize", "bwd_reduce", "bwd_dx"), ts):
        tot[k] = tot.get(k, 0.0) + t
    ssum = sum(ts)
    grand += ssum
    print(f"{li:5d} {str(s):>22} {4 * numel(s) / 1e6:7.1f} {ts[0]:7.1f} {ts[1]:7.1f} {ts[2]:7.1f} {ts[3]:7.1f} {ssum:8.1f} {32 * numel(s) / (ssum * 1e-6) / 1e9:9.0f}")
print("totals (us):", {k: round(v, 1) for k, v in tot.items()}, "sum", round(grand, 1))
