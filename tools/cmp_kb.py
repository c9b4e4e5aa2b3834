#!/usr/bin/env python3
"""Compare two kbench jsonl files (and optional bench lines): python tools/cmp_kb.py A B [benchA benchB]"""
import json
import sys


def load(f):
    out = {}
    for line in open(f):
        line = line.strip()
        if line.startswith("{"):
            d = json.loads(line)
            out[tuple(d["shape"])] = d
    return out


a, b = load(sys.argv[2]), load(sys.argv[1])
for k in a:
    row = [str(list(k))]
    for kern in ["fwd_stats", "bwd_reduce", "fwd_local", "bwd_local"]:
        if kern in a[k] and kern in b.get(k, {}):
            row.append(f"{kern} {b[k][kern]['us']:.2f}->{a[k][kern]['us']:.2f}")
    print("  ".join(row))
for f in sys.argv[3:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, round(d["value"]), round(d["ms_per_step"], 4),
          {k: round(v["ms_per_step"], 3) for k, v in d.get("kernels", {}).items()})
