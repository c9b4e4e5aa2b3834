#!/usr/bin/env python3
"""Producer-conv lab: per-layer device time of the tcgen05 conv (bf16 out, plain and with
the BN statistics epilogue) next to cuDNN's conv (torch conv2d, bf16 out), CUDA-graph
timed over rotating input sets (no L2 reuse between launches). One JSON line per layer.

    python tools/conv_lab.py [--layers all|3x3|small|c64] [--sets 3] [--iters 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import PRODUCER_LAYERS_NHWC  # noqa: E402
import paper_1711_07240_b200 as cg  # noqa: E402
from paper_1711_07240_b200 import producer as P  # noqa: E402


def timed(fn, iters, sets):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(iters):
            g.replay()
        e1.record(s)
        e1.synchronize()
    return e0.elapsed_time(e1) / iters / sets * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="all")
    ap.add_argument("--sets", type=int, default=3)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--batch", type=int, default=32)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cl = torch.channels_last
    layers = PRODUCER_LAYERS_NHWC
    if a.layers == "3x3":
        layers = [L for L in layers if L[0] == 3]
    elif a.layers == "small":
        layers = [L for L in layers if L[4] <= 14]
    elif a.layers == "c64":
        layers = [L for L in layers if L[3] <= 64]
    tot = {"ours": 0.0, "ours_stats": 0.0, "cudnn": 0.0}
    for k, sd, cin, cout, h, w, cnt in layers:
        xs = [torch.randn(a.batch, cin, h, w, device=dev).to(torch.bfloat16).contiguous(
            memory_format=cl) for _ in range(a.sets)]
        wt = (torch.randn(cout, cin, k, k, device=dev) / (k * k * cin) ** 0.5).to(
            torch.bfloat16).contiguous(memory_format=cl)
        conv = P.conv3x3 if k == 3 else P.conv1x1
        stats = P.conv3x3_stats if k == 3 else P.conv1x1_stats
        bf = torch.bfloat16
        t_o = timed(lambda: [conv(x, wt, stride=sd, out_dtype=bf) for x in xs], a.iters, a.sets)
        t_s = timed(lambda: [stats(x, wt, stride=sd, out_dtype=bf) for x in xs], a.iters, a.sets)
        # the statistics epilogue alone (slot table left in ws, no fold launch)
        t_sl = timed(lambda: [P._conv(x, wt, None, bf, k, True, sd, slots_only=True)
                              for x in xs], a.iters, a.sets)
        pad = k // 2
        t_c = timed(lambda: [torch.nn.functional.conv2d(x, wt, stride=sd, padding=pad)
                             for x in xs], a.iters, a.sets)
        # the producer fusion itself: fused conv + BN forward vs cuDNN conv + our BN forward
        sts = [cg.BNLayerState.create(cout, device=dev) for _ in range(a.sets)]
        fused = P.conv3x3_bn_forward_local if k == 3 else P.conv1x1_bn_forward_local
        t_f = timed(lambda: [fused(x, wt, st, stride=sd, out_dtype=bf) for x, st in zip(xs, sts)],
                    a.iters, a.sets)
        t_cs = timed(lambda: [cg.bn_forward_local(torch.nn.functional.conv2d(
            x, wt, stride=sd, padding=pad), st) for x, st in zip(xs, sts)], a.iters, a.sets)
        # parity of the plain conv against cuDNN's (both bf16 out)
        z = conv(xs[0], wt, stride=sd, out_dtype=bf).float()
        zr = torch.nn.functional.conv2d(xs[0], wt, stride=sd, padding=pad).float()
        err = ((z - zr).abs().max() / zr.abs().max()).item()
        flops = 2.0 * a.batch * (h // sd) * (w // sd) * cout * cin * k * k
        print(json.dumps({"k": k, "stride": sd, "cin": cin, "cout": cout, "hw": h, "count": cnt,
                          "ours_us": round(t_o, 2), "ours_stats_us": round(t_s, 2),
                          "ours_slots_us": round(t_sl, 2), "fused_us": round(t_f, 2),
                          "cudnn_split_us": round(t_cs, 2),
                          "cudnn_us": round(t_c, 2), "ours_tflops": round(flops / t_o / 1e6),
                          "cudnn_tflops": round(flops / t_c / 1e6),
                          "ratio": round(t_c / t_o, 3), "rel_err": err}), flush=True)
        tot["ours"] += cnt * t_o
        tot["ours_stats"] += cnt * t_s
        tot["cudnn"] += cnt * t_c
        tot["fused"] = tot.get("fused", 0.0) + cnt * t_f
        tot["cudnn_split"] = tot.get("cudnn_split", 0.0) + cnt * t_cs
        tot["slots"] = tot.get("slots", 0.0) + cnt * t_sl
        del xs
    print(json.dumps({"total_us": {k: round(v, 1) for k, v in tot.items()},
                      "ratio": round(tot["cudnn"] / tot["ours"], 3),
                      "fused_vs_cudnn_split": round(tot["cudnn_split"] / tot["fused"], 3)}),
          flush=True)


if __name__ == "__main__":
    main()
