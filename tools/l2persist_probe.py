#!/usr/bin/env python3
"""Probe: does an L2 persisting access-policy window over [x | dy] let the backward's dx
pass re-read x and dy from L2 after the backward reduction read them?

For each shape: forward once (public API), flush L2, then time bn_backward_local (bwd
reduce + dx) with CUDA events on the launch stream, without and with a persisting window
(driver API cuStreamSetAttribute). Persisting lines are reset and L2 flushed before every
timed iteration, so each iteration starts cold; a device sleep ahead of the first event
lets the host enqueue the whole backward, so the events see device time only.

    python tools/l2persist_probe.py [--iters 20]
"""

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1711_07240_b200 as cg  # noqa: E402

cu = ctypes.CDLL("libcuda.so.1")
CU_LIMIT_PERSISTING_L2_CACHE_SIZE = 0x06
CU_DEVICE_ATTRIBUTE_MAX_PERSISTING_L2_CACHE_SIZE = 108
CU_DEVICE_ATTRIBUTE_MAX_ACCESS_POLICY_WINDOW_SIZE = 109
CU_STREAM_ATTRIBUTE_ACCESS_POLICY_WINDOW = 1


class Window(ctypes.Structure):
    _fields_ = [("base_ptr", ctypes.c_void_p), ("num_bytes", ctypes.c_size_t),
                ("hitRatio", ctypes.c_float), ("hitProp", ctypes.c_int),
                ("missProp", ctypes.c_int), ("_pad", ctypes.c_byte * 36)]


def attr(a):
    v = ctypes.c_int()
    assert cu.cuDeviceGetAttribute(ctypes.byref(v), a, 0) == 0
    return v.value


def set_window(stream, ptr, nbytes, ratio):
    w = Window()
    w.base_ptr = ptr
    w.num_bytes = nbytes
    w.hitRatio = ratio
    w.hitProp = 2 if nbytes else 0  # persisting / normal
    w.missProp = 1 if nbytes else 0  # streaming
    rc = cu.cuStreamSetAttribute(ctypes.c_void_p(stream), CU_STREAM_ATTRIBUTE_ACCESS_POLICY_WINDOW,
                                 ctypes.byref(w))
    assert rc == 0, rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    torch.zeros(1, device=dev)
    cg.set_strict(False)  # no per-call status sync (as in bench.py)
    pmax, wmax = attr(CU_DEVICE_ATTRIBUTE_MAX_PERSISTING_L2_CACHE_SIZE), attr(
        CU_DEVICE_ATTRIBUTE_MAX_ACCESS_POLICY_WINDOW_SIZE)
    assert cu.cuCtxSetLimit(CU_LIMIT_PERSISTING_L2_CACHE_SIZE, ctypes.c_size_t(pmax)) == 0
    print(json.dumps({"max_persisting_l2": pmax, "max_window": wmax}), flush=True)
    flush = torch.empty(512 * 2**20 // 4, device=dev)
    stream = torch.cuda.current_stream()
    for shape in [(32, 64, 56, 56), (32, 128, 28, 28), (32, 512, 28, 28), (32, 1024, 14, 14), (32, 256, 56, 56),
                  (32, 64, 112, 112)]:
        e = shape[0] * shape[1] * shape[2] * shape[3]
        buf = torch.randn(2 * e, device=dev)
        x, dy = buf[:e].view(shape), buf[e:].view(shape)
        st = cg.BNLayerState(gamma=torch.ones(shape[1]), beta=torch.zeros(shape[1]))
        _, cache = cg.bn_forward_local(x, st)
        nbytes = 8 * e
        row = {"shape": list(shape), "bytes_x_dy": nbytes}
        for name, win in [("base", 0), ("persist", min(nbytes, wmax)), ("base2", 0)]:
            ratio = min(1.0, pmax / win) if win else 0.0
            ts = []
            for _ in range(args.iters):
                set_window(stream.cuda_stream, 0, 0, 0.0)
                cu.cuCtxResetPersistingL2Cache()
                flush.zero_()
                set_window(stream.cuda_stream, buf.data_ptr() if win else 0, win, ratio)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(3_000_000)  # the host enqueues the step while the GPU waits
                a.record(stream)
                cg.bn_backward_local(dy, cache, st)
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            ts.sort()
            row[name + "_us"] = round(ts[len(ts) // 2], 2)
            row[name + "_ratio"] = round(ratio, 3)
        set_window(stream.cuda_stream, 0, 0, 0.0)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
