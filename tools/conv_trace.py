#!/usr/bin/env python3
"""Per-(CTA, work unit) timeline of one producer-conv launch from globaltimer stamps
(debug hook cgbn_debug_conv_trace): producer start, MMA done (tfull committed), epilogue
has the accumulator, split-K hand-off done (release / wait), epilogue done.

    CGBN_CONV_SPLITS=2 python tools/conv_trace.py --layer 1,1,1024,256,14   # k,s,cin,cout,hw
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_07240_b200 import _lib  # noqa: E402
from paper_1711_07240_b200 import producer as P  # noqa: E402

EV = ["prod_start", "mma_done", "epi_acc", "handoff", "epi_done", "-", "-", "partials_added"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="1,1,1024,256,14")
    ap.add_argument("--batch", type=int, default=32)
    a = ap.parse_args()
    k, sd, cin, cout, hw = (int(v) for v in a.layer.split(","))
    dev = torch.device("cuda", 0)
    x = torch.randn(a.batch, cin, hw, hw, device=dev).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    wt = (torch.randn(cout, cin, k, k, device=dev) / (k * k * cin) ** 0.5).to(
        torch.bfloat16).contiguous(memory_format=torch.channels_last)
    conv = P.conv3x3 if k == 3 else P.conv1x1
    for _ in range(3):
        conv(x, wt, stride=sd, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    lib = _lib.load()
    hook = lib.cgbn_debug_conv_trace
    hook.argtypes = [ctypes.c_void_p]
    tr = torch.zeros(160 * 16 * 8, dtype=torch.int64, device=dev)
    hook(tr.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    conv(x, wt, stride=sd, out_dtype=torch.bfloat16)
    e1.record()
    torch.cuda.synchronize()
    hook(None)
    t = tr.view(160, 16, 8).cpu().numpy().astype(np.int64)
    used = t[:, :, 0] > 0
    t0 = t[:, :, 0][used].min()
    out = {"layer": a.layer, "event_us": round(e0.elapsed_time(e1) * 1e3, 2),
           "ctas": int(used.any(axis=1).sum()), "units_max": int(used.sum(axis=1).max())}
    for li in range(int(used.sum(axis=1).max())):
        rows = t[:, li][used[:, li]]
        rec = {}
        for j, name in enumerate(EV):
            if name == "-":
                continue
            col = rows[:, j]
            col = col[col > 0]
            if len(col):
                rec[name] = [round(float(np.percentile((col - t0) / 1e3, p)), 2) for p in (0, 50, 100)]
        fin = rows[:, 6]
        rec["splits_seen"] = sorted(set(int(v) for v in fin))
        out[f"unit{li}"] = rec
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
