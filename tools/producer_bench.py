"""Producer-fusion measurements on the ResNet-50 1x1-conv -> BN
layers at batch 32 (H*W a multiple of 8: layer1 56x56 and layer2 28x28; the stride-2
downsample is excluded).

Per layer and output dtype, CUDA-graph timed (3 buffer sets rotated inside the graph so
consecutive launches never find their operands in L2):
  conv        our tcgen05 conv1x1 alone                     GB/s = (x + w + z bytes) / t
  conv_stats  conv1x1 + epilogue partial + fold
  fused_fwd   conv1x1_bn_forward_local (conv+stats, finalize, normalise)
  split_fwd   conv1x1 then bn_forward_local(z) (statistics kernel re-reads z)
  cudnn_fwd   torch conv2d (cuDNN, bf16 out only) then bn_forward_local(z)
Prints one JSON line per (layer, dtype).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1711_07240_b200 as cg  # noqa: E402
from paper_1711_07240_b200 import producer as P  # noqa: E402

LAYERS_NHWC = [  # (name, k, Cin, Cout, H, W, count in ResNet-50): channels_last producers
    ("l1.conv2", 3, 64, 64, 56, 56, 3),
    ("l2.conv2", 3, 128, 128, 28, 28, 3),
    ("l3.conv2", 3, 256, 256, 14, 14, 5),
    ("l4.conv2", 3, 512, 512, 7, 7, 2),
    ("l1.conv3", 1, 64, 256, 56, 56, 3),
    ("l2.conv3", 1, 128, 512, 28, 28, 4),
    ("l3.conv1", 1, 1024, 256, 14, 14, 5),
    ("l3.conv3", 1, 256, 1024, 14, 14, 6),
    ("l4.conv3", 1, 512, 2048, 7, 7, 3),
]

LAYERS = [  # (name, Cin, Cout, H, W, count in ResNet-50)
    ("l1.conv1.first", 64, 64, 56, 56, 1),
    ("l1.conv1", 256, 64, 56, 56, 2),
    ("l1.conv3", 64, 256, 56, 56, 3),
    ("l1.down", 64, 256, 56, 56, 1),
    ("l2.conv1.first", 256, 128, 56, 56, 1),
    ("l2.conv1", 512, 128, 28, 28, 3),
    ("l2.conv3", 128, 512, 28, 28, 4),
]


def timed(fn, iters=20, warm=3):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(iters):
            g.replay()
        e1.record(s)
        e1.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us per graph replay


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--sets", type=int, default=3)
    ap.add_argument("--layers", default="")
    ap.add_argument("--layout", choices=["nchw", "nhwc"], default="nchw")
    args = ap.parse_args()
    if args.layout == "nhwc":
        return main_nhwc(args)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cg.set_strict(False)
    peak = 6549.8
    for name, cin, cout, h, w, cnt in LAYERS:
        if args.layers and name not in args.layers.split(","):
            continue
        n = args.batch
        K = args.sets
        xs = [torch.randn(n, cin, h, w, device=dev).to(torch.bfloat16) for _ in range(K)]
        wt = (torch.randn(cout, cin, device=dev) / cin ** 0.5).to(torch.bfloat16)
        w4 = wt.view(cout, cin, 1, 1)
        for od in (torch.float32, torch.bfloat16):
            sts = [cg.BNLayerState.create(cout, device=dev) for _ in range(K)]
            esz = 4 if od == torch.float32 else 2
            e = n * cout * h * w
            conv_bytes = n * cin * h * w * 2 + cout * cin * 2 + e * esz
            zs = [P.conv1x1(x, wt, out_dtype=od) for x in xs]
            res = {"layer": name, "N": n, "Cin": cin, "Cout": cout, "HW": [h, w], "count": cnt,
                   "z_dtype": str(od).replace("torch.", ""), "conv_bytes": conv_bytes}

            def conv():
                for x in xs:
                    P.conv1x1(x, wt, out_dtype=od)

            def conv_stats():
                for x in xs:
                    P.conv1x1_stats(x, wt, out_dtype=od)

            def fused():
                for x, st in zip(xs, sts):
                    P.conv1x1_bn_forward_local(x, wt, st, out_dtype=od)

            def split():
                for x, st in zip(xs, sts):
                    z = P.conv1x1(x, wt, out_dtype=od)
                    cg.bn_forward_local(z, st)

            def bn_only():
                for z, st in zip(zs, sts):
                    cg.bn_forward_local(z, st)

            res["conv_us"] = timed(conv) / K
            res["conv_gbs"] = conv_bytes / res["conv_us"] / 1e3
            res["conv_hbm_frac"] = res["conv_gbs"] / peak
            res["conv_stats_us"] = timed(conv_stats) / K
            res["fused_fwd_us"] = timed(fused) / K
            res["split_fwd_us"] = timed(split) / K
            res["bn_fwd_only_us"] = timed(bn_only) / K
            res["fused_fwd_bytes"] = conv_bytes + 2 * e * esz
            res["fused_fwd_gbs"] = res["fused_fwd_bytes"] / res["fused_fwd_us"] / 1e3
            if od == torch.bfloat16:
                def cudnn():
                    for x, st in zip(xs, sts):
                        z = torch.nn.functional.conv2d(x, w4)
                        cg.bn_forward_local(z, st)

                def cudnn_conv():
                    for x in xs:
                        torch.nn.functional.conv2d(x, w4)
                res["cudnn_conv_us"] = timed(cudnn_conv) / K
                res["cudnn_fwd_us"] = timed(cudnn) / K
            res["speedup_fused_vs_split"] = res["split_fwd_us"] / res["fused_fwd_us"]
            print(json.dumps(res), flush=True)


def main_nhwc(args):
    """channels_last producers (1x1 and 3x3): fused vs split BN forward, vs cuDNN."""
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cg.set_strict(False)
    peak = 6549.8
    cl = torch.channels_last
    for name, k, cin, cout, h, w, cnt in LAYERS_NHWC:
        if args.layers and name not in args.layers.split(","):
            continue
        n, K = args.batch, args.sets
        xs = [torch.randn(n, cin, h, w, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
              for _ in range(K)]
        wt = (torch.randn(cout, cin, k, k, device=dev) / (k * k * cin) ** 0.5).to(torch.bfloat16)
        conv = P.conv3x3 if k == 3 else P.conv1x1
        fused_fn = P.conv3x3_bn_forward_local if k == 3 else P.conv1x1_bn_forward_local
        for od in (torch.float32, torch.bfloat16):
            sts = [cg.BNLayerState.create(cout, device=dev) for _ in range(K)]
            esz = 4 if od == torch.float32 else 2
            e = n * cout * h * w
            conv_bytes = n * cin * h * w * 2 + cout * cin * k * k * 2 + e * esz
            flops = 2.0 * e * cin * k * k
            res = {"layer": name, "k": k, "N": n, "Cin": cin, "Cout": cout, "HW": [h, w],
                   "count": cnt, "z_dtype": str(od).replace("torch.", ""), "layout": "NHWC"}
            res["conv_us"] = timed(lambda: [conv(x, wt, out_dtype=od) for x in xs]) / K
            res["conv_hbm_frac"] = conv_bytes / res["conv_us"] / 1e3 / peak
            res["conv_tflops"] = flops / res["conv_us"] / 1e6
            res["fused_fwd_us"] = timed(lambda: [fused_fn(x, wt, st, out_dtype=od)
                                                 for x, st in zip(xs, sts)]) / K
            res["split_fwd_us"] = timed(lambda: [cg.bn_forward_local(conv(x, wt, out_dtype=od), st)
                                                 for x, st in zip(xs, sts)]) / K
            if od == torch.bfloat16:
                pad = 1 if k == 3 else 0
                res["cudnn_conv_us"] = timed(
                    lambda: [torch.nn.functional.conv2d(x, wt, padding=pad) for x in xs]) / K
                res["cudnn_fwd_us"] = timed(
                    lambda: [cg.bn_forward_local(torch.nn.functional.conv2d(x, wt, padding=pad), st)
                             for x, st in zip(xs, sts)]) / K
            res["speedup_fused_vs_split"] = res["split_fwd_us"] / res["fused_fwd_us"]
            print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    main()
