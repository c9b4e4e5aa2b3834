"""Host cost of the eager public API per layout / dtype: wall time of enqueueing one
ResNet-50 step (53 sync_bn_forward + 53 sync_bn_backward) vs its device time."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1711_07240_b200 as cg  # noqa: E402

dev = torch.device("cuda", 0)
shapes = bench.resnet50_bn_shapes(32)
h = cg.SoloHandle(dev)
for layout, act in (("nchw", torch.float32), ("nhwc", torch.float32), ("nhwc", torch.bfloat16)):
    mf = torch.channels_last if layout == "nhwc" else torch.contiguous_format
    xs = [torch.randn(s, device=dev).to(act).contiguous(memory_format=mf) for s in shapes]
    dys = [torch.randn(s, device=dev).to(act).contiguous(memory_format=mf) for s in shapes]
    sts = [cg.BNLayerState(gamma=torch.rand(s[1], device=dev) + 0.5,
                           beta=torch.randn(s[1], device=dev)) for s in shapes]

    def step():
        caches = [cg.sync_bn_forward(h, x, st)[1] for x, st in zip(xs, sts)]
        for i in range(len(xs) - 1, -1, -1):
            cg.sync_bn_backward(h, dys[i], caches[i], sts[i])

    step()
    torch.cuda.synchronize()
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        step()
        t_host = time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
        print(f"{layout} {act}: host enqueue {t_host * 1e3:.1f} ms, device {e0.elapsed_time(e1):.1f} ms",
              flush=True)
    del xs, dys
