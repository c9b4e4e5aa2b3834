#!/usr/bin/env python3
"""Side-by-side table of conv_lab.py runs: python tools/conv_cmp.py name=file.jsonl ..."""
import json
import sys

runs = [(a.split("=", 1)[0], [json.loads(l) for l in open(a.split("=", 1)[1])]) for a in sys.argv[1:]]
n = len(runs[0][1]) - 1
print("k s  cin cout hw cnt | " + " ".join(f"{k:>8}" for k, _ in runs) + " |  cudnn | slots: " +
      " ".join(k for k, _ in runs) + " | fused: " + " ".join(k for k, _ in runs) + " | cudnn+bn")
for i in range(n):
    p = runs[0][1][i]
    print(f"{p['k']} {p['stride']} {p['cin']:4d} {p['cout']:4d} {p['hw']:3d} {p['count']:2d} | " +
          " ".join(f"{r[i]['ours_us']:8.2f}" for _, r in runs) + f" | {p['cudnn_us']:6.2f} | " +
          " ".join(f"{r[i].get('ours_slots_us', 0):6.2f}" for _, r in runs) + " | " +
          " ".join(f"{r[i].get('fused_us', 0):6.2f}" for _, r in runs) +
          f" | {p.get('cudnn_split_us', 0):6.2f}")
for k, r in runs:
    print(k, r[-1])
