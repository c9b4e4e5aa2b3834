#!/usr/bin/env python3
"""Per-layer / per-kernel device times of one bench step from an ncu launch list
(gpu__time_duration.sum + dram bytes), taken with
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --cache-control none --csv --log-file L.csv \
        python bench.py --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-kprof
The last 4*53 CGBN launches of the list are the measured step (fwd: reduce, elementwise
per layer; bwd: reduce, elementwise per layer in reverse order)."""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import numel, resnet50_bn_shapes  # noqa: E402


def load_step(path):
    """The measured step's 4*53 launches: (fwd, bwd) lists of per-launch metric dicts."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    k = {}
    for r in rows[1:]:
        d = k.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    ours = [k[i] for i in sorted(k) if ("k_reduce" in k[i]["name"] or "k_ew" in k[i]["name"])]
    shapes = resnet50_bn_shapes(32)
    step = ours[-4 * len(shapes):]
    return shapes, step[:2 * len(shapes)], step[2 * len(shapes):]


def traffic_json(path, out):
    """Per-family dram bytes per launch (what bench.py reports as roofline.traffic)."""
    shapes, fwd, bwd = load_step(path)
    fam = {"fwd_stats": [], "fwd_normalize_ew": [], "bwd_reduce": [], "bwd_dx": []}
    bpe = {"fwd_stats": 4, "fwd_normalize_ew": 8, "bwd_reduce": 8, "bwd_dx": 12}
    for li, s in enumerate(shapes):
        bi = len(shapes) - 1 - li
        for name, kk in zip(fam, (fwd[2 * li], fwd[2 * li + 1], bwd[2 * bi], bwd[2 * bi + 1])):
            fam[name].append((kk, numel(s)))
    res = {}
    tot_t = sum(kk["gpu__time_duration.sum"] for v in fam.values() for kk, _ in v)
    for name, v in fam.items():
        n = len(v)
        dram = sum(kk.get("dram__bytes_read.sum", 0) + kk.get("dram__bytes_write.sum", 0)
                   for kk, _ in v)
        alg = sum(bpe[name] * e for _, e in v)
        t = sum(kk["gpu__time_duration.sum"] for kk, _ in v)
        res[name] = {"launches": n, "dram_bytes_per_launch": dram / n,
                     "alg_bytes_per_launch": alg / n, "dram_over_alg": dram / alg,
                     "ncu_time_us_per_step": t / 1e3, "ncu_share": t / tot_t}
    doc = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                     "dram__bytes_write.sum --cache-control none --clock-control none on "
                     "`python bench.py --steps 1 --warmup 3 --no-graph --no-e2e "
                     "--no-cpu-baseline --no-kprof` (one eager step; per-kernel-family sums "
                     "over the 53 layers). Per-launch dram bytes include write-backs of "
                     "lines the previous kernel left dirty in L2.",
           "launch_list": os.path.basename(path), "families": res}
    import json
    json.dump(doc, open(out, "w"), indent=1)


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    k = {}
    for r in rows[1:]:
        d = k.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    ours = [k[i] for i in sorted(k) if ("k_reduce" in k[i]["name"] or "k_ew" in k[i]["name"])]
    shapes = resnet50_bn_shapes(32)
    step = ours[-4 * len(shapes):]
    fwd, bwd = step[:2 * len(shapes)], step[2 * len(shapes):]
    print(f"{'l':>3} {'C,H,W':>16} {'stats':>6} {'norm':>6} {'bred':>6} {'dx':>6} {'sum us':>7}"
          f" {'alg GB/s':>8} {'dram/alg':>8}")
    tot = [0.0] * 4
    dram = alg = 0.0
    for li, s in enumerate(shapes):
        bi = len(shapes) - 1 - li
        ks = (fwd[2 * li], fwd[2 * li + 1], bwd[2 * bi], bwd[2 * bi + 1])
        t = [x["gpu__time_duration.sum"] / 1e3 for x in ks]
        by = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in ks)
        for i in range(4):
            tot[i] += t[i]
        dram += by
        alg += 32 * numel(s)
        print(f"{li:3d} {str(s[1:]):>16} {t[0]:6.1f} {t[1]:6.1f} {t[2]:6.1f} {t[3]:6.1f} "
              f"{sum(t):7.1f} {32 * numel(s) / (sum(t) * 1e-6) / 1e9:8.0f} {by / (32 * numel(s)):8.2f}")
    print("totals us: stats %.1f norm %.1f bred %.1f dx %.1f | sum %.1f | dram/alg %.3f"
          % (tot[0], tot[1], tot[2], tot[3], sum(tot), dram / alg))


if __name__ == "__main__":
    if len(sys.argv) > 3 and sys.argv[2] == "--traffic":
        traffic_json(sys.argv[1], sys.argv[3])
    else:
        main(sys.argv[1])
