#!/usr/bin/env python3
"""Per-kernel microbenchmark of the CGBN C ABI (used for roofline work and ncu runs).

For each shape, every kernel (fwd_stats, fwd_normalize, bwd_reduce, bwd_dx) is launched
through the C ABI on rotating buffer sets whose total exceeds 2x the L2 (so each
launch reads from HBM), timed with CUDA events on the launch stream, and reported as
algorithmic GB/s (stats 4, normalize 8, bwd_reduce 8, bwd_dx 12 B/elem).

    python tools/kbench.py --shape 32,256,56,56 --shape 32,2048,7,7 [--iters 50]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1711_07240_b200 import _lib  # noqa: E402

L2_BYTES = 126 * 1024 * 1024


def run_shape(shape, iters, layout, relu, graph=False, dtype=torch.float32):
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    st0 = torch.cuda.current_stream().cuda_stream
    nonlocal_st = [st0]
    st = st0
    n, c, h, w = shape
    hw = h * w
    e = n * c * hw
    per_set = 16 * e  # x, dy, y, dx
    sets = max(2, int(-(-2 * L2_BYTES // per_set)) + 1)
    sets = min(sets, 64)
    bufs = []
    for _ in range(sets):
        x = torch.randn(shape, device=dev).to(dtype)
        dy = torch.randn(shape, device=dev).to(dtype)
        if (layout & 0xF) == _lib.LAYOUT_NHWC:
            x = x.contiguous(memory_format=torch.channels_last)
            dy = dy.contiguous(memory_format=torch.channels_last)
        bufs.append((x, dy, torch.empty_like(x), torch.empty_like(x)))
    gamma = torch.rand(c, device=dev) + 0.5
    beta = torch.randn(c, device=dev)
    rm = torch.zeros(c, device=dev)
    rv = torch.ones(c, device=dev)
    part = torch.empty(2 * c + 1, dtype=torch.float64, device=dev)
    bpart = torch.empty(2 * c, dtype=torch.float64, device=dev)
    saved = torch.empty(3 * c + 1, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    nb = lib.cgbn_workspace_bytes(n, c, hw, layout)
    ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)
    pa, keep1 = _lib.ptr_array([part.data_ptr()])
    pb, keep2 = _lib.ptr_array([bpart.data_ptr()])
    dg = torch.empty(c, device=dev)
    db = torch.empty(c, device=dev)

    def k_stats(b):
        return lib.cgbn_fwd_stats(b[0].data_ptr(), n, c, hw, layout, part.data_ptr(),
                                  ws.data_ptr(), ws.numel(), nonlocal_st[0])

    def k_norm(b):
        return lib.cgbn_fwd_normalize(b[0].data_ptr(), n, c, hw, layout, pa, 1,
                                      gamma.data_ptr(), beta.data_ptr(), 1e-5, 0.1,
                                      rm.data_ptr(), rv.data_ptr(), saved.data_ptr(), int(relu),
                                      b[2].data_ptr(), status.data_ptr(), ws.data_ptr(),
                                      ws.numel(), nonlocal_st[0])

    def k_bred(b):
        return lib.cgbn_bwd_reduce(b[1].data_ptr(), b[0].data_ptr(), n, c, hw, layout,
                                   saved.data_ptr(), gamma.data_ptr(), beta.data_ptr(), int(relu),
                                   bpart.data_ptr(), ws.data_ptr(), ws.numel(), nonlocal_st[0])

    def k_dx(b):
        return lib.cgbn_bwd_dx(b[1].data_ptr(), b[0].data_ptr(), n, c, hw, layout, pb, 1,
                               saved.data_ptr(), gamma.data_ptr(), beta.data_ptr(), 1e-5,
                               int(relu), b[3].data_ptr(), dg.data_ptr(), db.data_ptr(),
                               status.data_ptr(), ws.data_ptr(), ws.numel(), nonlocal_st[0])

    def k_lfwd(b):
        return lib.cgbn_fwd_train_local(b[0].data_ptr(), n, c, hw, layout, gamma.data_ptr(),
                                        beta.data_ptr(), 1e-5, 0.1, rm.data_ptr(), rv.data_ptr(),
                                        saved.data_ptr(), int(relu), b[2].data_ptr(),
                                        status.data_ptr(), ws.data_ptr(), ws.numel(), nonlocal_st[0])

    def k_lbwd(b):
        return lib.cgbn_bwd_local(b[1].data_ptr(), b[0].data_ptr(), n, c, hw, layout,
                                  saved.data_ptr(), gamma.data_ptr(), beta.data_ptr(), 1e-5,
                                  int(relu), b[3].data_ptr(), dg.data_ptr(), db.data_ptr(),
                                  status.data_ptr(), ws.data_ptr(), ws.numel(), nonlocal_st[0])

    def k_ffwd(b):
        return lib.cgbn_fwd_fused(b[0].data_ptr(), n, c, hw, layout, gamma.data_ptr(),
                                  beta.data_ptr(), 1e-5, 0.1, rm.data_ptr(), rv.data_ptr(),
                                  saved.data_ptr(), int(relu), b[2].data_ptr(), status.data_ptr(),
                                  ws.data_ptr(), ws.numel(), nonlocal_st[0])

    def k_fbwd(b):
        return lib.cgbn_bwd_fused(b[1].data_ptr(), b[0].data_ptr(), n, c, hw, layout,
                                  saved.data_ptr(), gamma.data_ptr(), beta.data_ptr(), 1e-5,
                                  int(relu), b[3].data_ptr(), dg.data_ptr(), db.data_ptr(),
                                  status.data_ptr(), ws.data_ptr(), ws.numel(), nonlocal_st[0])

    out = {"shape": list(shape), "elements": e, "rotating_sets": sets}
    kernels = [("fwd_stats", k_stats, 4), ("fwd_normalize", k_norm, 8),
               ("bwd_reduce", k_bred, 8), ("bwd_dx", k_dx, 12),
               ("fwd_local", k_lfwd, 12), ("bwd_local", k_lbwd, 20)]
    if lib.cgbn_fused_supported(n, c, hw, layout, 0):
        kernels.append(("fwd_fused", k_ffwd, 12))
    if lib.cgbn_fused_supported(n, c, hw, layout, 1):
        kernels.append(("bwd_fused", k_fbwd, 20))
    for name, fn, bpe in kernels:
        for i in range(3):
            _lib.check(fn(bufs[i % sets]), name)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if graph:
            gr = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                gst = side.cuda_stream
                nonlocal_st[0] = gst
                with torch.cuda.graph(gr, stream=side):
                    for i in range(iters):
                        fn(bufs[i % sets])
                nonlocal_st[0] = st
            torch.cuda.current_stream().wait_stream(side)
            gr.replay()
            torch.cuda.synchronize()
            e0.record()
            gr.replay()
            e1.record()
        else:
            e0.record()
            for i in range(iters):
                fn(bufs[i % sets])
            e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
        esz = torch.finfo(dtype).bits // 8
        out[name] = {"us": round(us, 2),
                     "alg_gbs": round(bpe * esz / 4 * e / (us * 1e-6) / 1e9, 1)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", action="append", default=[])
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--nhwc", action="store_true")
    ap.add_argument("--relu", action="store_true")
    ap.add_argument("--graph", action="store_true", help="time inside a CUDA graph")
    ap.add_argument("--dtype", choices=["f32", "bf16", "f16"], default="f32",
                    help="activation dtype (bytes per element scale the GB/s)")
    args = ap.parse_args()
    shapes = [tuple(int(v) for v in s.split(",")) for s in args.shape] or [
        (32, 64, 112, 112), (32, 256, 56, 56), (32, 64, 56, 56), (32, 512, 28, 28),
        (32, 128, 28, 28), (32, 1024, 14, 14), (32, 256, 14, 14), (32, 2048, 7, 7),
        (32, 512, 7, 7), (2, 256, 200, 334), (2, 64, 400, 667), (1, 2048, 7, 7)]
    layout = _lib.LAYOUT_NHWC if args.nhwc else _lib.LAYOUT_NCHW
    dtype, act = {"f32": (torch.float32, _lib.ACT_F32), "bf16": (torch.bfloat16, _lib.ACT_BF16),
                  "f16": (torch.float16, _lib.ACT_F16)}[args.dtype]
    for s in shapes:
        r = run_shape(s, args.iters, layout | act, args.relu, args.graph, dtype)
        r["dtype"] = args.dtype
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
