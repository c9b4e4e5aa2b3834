"""One plain conv / conv+statistics launch pair (after warm-up) for ncu captures.

    python tools/conv_once.py N,Cin,Cout,H,W [f32|bf16] [nchw1|nhwc1|nhwc3]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_07240_b200 import producer as P  # noqa: E402

n, cin, cout, h, w = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32,64,64,56,56").split(",")]
od = torch.bfloat16 if len(sys.argv) > 2 and sys.argv[2] == "bf16" else torch.float32
mode = sys.argv[3] if len(sys.argv) > 3 else "nchw1"
dev = torch.device("cuda", 0)
x = torch.randn(n, cin, h, w, device=dev).to(torch.bfloat16)
k = 3 if mode == "nhwc3" else 1
wt = (torch.randn(cout, cin, k, k, device=dev) / (k * k * cin) ** 0.5).to(torch.bfloat16)
if mode != "nchw1":
    x = x.contiguous(memory_format=torch.channels_last)
conv = P.conv3x3 if k == 3 else P.conv1x1
stats = P.conv3x3_stats if k == 3 else P.conv1x1_stats
for _ in range(3):
    conv(x, wt, out_dtype=od)
    stats(x, wt, out_dtype=od)
torch.cuda.synchronize()
conv(x, wt, out_dtype=od)
stats(x, wt, out_dtype=od)
torch.cuda.synchronize()
print("ok")
