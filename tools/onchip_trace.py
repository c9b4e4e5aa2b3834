#!/usr/bin/env python3
"""Phase timing of the on-chip BN kernels (cgbn_onchip.cuh) from per-CTA globaltimer
stamps (debug hook cgbn_debug_onchip_trace_a0, fp32 unit): launch -> after PDL wait ->
copies issued -> all copies landed -> reduction + cluster barrier -> finisher -> end.

    python tools/onchip_trace.py --shape 32,128,28,28 [--force nch,kc]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_07240_b200 import _lib  # noqa: E402

PH = ["start", "pdl_wait", "issued", "setup", "reduced", "finished", "written"]


def run(shape, bwd, reps=3):
    lib = _lib.load()
    hook = lib.cgbn_debug_onchip_trace_a0
    hook.argtypes = [ctypes.c_void_p]
    dev = torch.device("cuda", 0)
    n, c, h, w = shape
    x = torch.randn(shape, device=dev)
    dy = torch.randn(shape, device=dev)
    y = torch.empty_like(x)
    gamma = torch.rand(c, device=dev) + 0.5
    beta = torch.randn(c, device=dev)
    rm, rv = torch.zeros(c, device=dev), torch.ones(c, device=dev)
    saved = torch.empty(3 * c + 1, dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.zeros(lib.cgbn_workspace_bytes(n, c, h * w, 0), dtype=torch.uint8, device=dev)
    dg, db = torch.empty(c, device=dev), torch.empty(c, device=dev)
    tr = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def fwd():
        return lib.cgbn_fwd_fused(x.data_ptr(), n, c, h * w, 0, gamma.data_ptr(),
                                  beta.data_ptr(), 1e-5, 0.1, rm.data_ptr(), rv.data_ptr(),
                                  saved.data_ptr(), 0, y.data_ptr(), status.data_ptr(),
                                  ws.data_ptr(), ws.numel(), st)

    def bwdf():
        return lib.cgbn_bwd_fused(dy.data_ptr(), x.data_ptr(), n, c, h * w, 0, saved.data_ptr(),
                                  gamma.data_ptr(), beta.data_ptr(), 1e-5, 0, y.data_ptr(),
                                  dg.data_ptr(), db.data_ptr(), status.data_ptr(),
                                  ws.data_ptr(), ws.numel(), st)

    _lib.check(fwd(), "fwd")
    fn = bwdf if bwd else fwd
    for _ in range(reps):
        _lib.check(fn(), "onchip")
    torch.cuda.synchronize()
    hook(tr.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(fn(), "onchip")
    e1.record()
    torch.cuda.synchronize()
    hook(None)
    t = tr.view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = (t[:, :12] - t0) / 1e3  # us
    out = {"shape": list(shape), "dir": "bwd" if bwd else "fwd", "ctas": int(len(t)),
           "event_us": e0.elapsed_time(e1) * 1e3, "span_us": float(rel[:, 6].max()),
           "ctas_per_sm_max": int(np.bincount(t[:, 15].astype(int)).max())}
    for q in range(4):
        col = rel[:, 8 + q][t[:, 8 + q] > 0]
        if len(col):
            out[f"group{q}"] = [round(float(np.percentile(col, v)), 2) for v in (0, 50, 100)]
    for k, name in enumerate(PH):
        col = rel[:, k]
        out[name] = [round(float(np.percentile(col, q)), 2) for q in (0, 50, 100)]
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", action="append", default=[])
    a = ap.parse_args()
    shapes = [tuple(int(v) for v in s.split(",")) for s in a.shape] or [(32, 128, 28, 28)]
    for s in shapes:
        for bwd in (False, True):
            print(json.dumps(run(s, bwd)), flush=True)
