"""One conv1x1 / conv1x1_stats launch pair (after warm-up) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1711_07240_b200 import producer as P
n, cin, cout, h, w = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32,64,64,56,56").split(",")]
od = torch.bfloat16 if len(sys.argv) > 2 and sys.argv[2] == "bf16" else torch.float32
dev = torch.device("cuda", 0)
x = torch.randn(n, cin, h, w, device=dev).to(torch.bfloat16)
wt = (torch.randn(cout, cin, device=dev) / cin ** 0.5).to(torch.bfloat16)
for _ in range(3):
    P.conv1x1(x, wt, out_dtype=od)
    P.conv1x1_stats(x, wt, out_dtype=od)
torch.cuda.synchronize()
P.conv1x1(x, wt, out_dtype=od)
P.conv1x1_stats(x, wt, out_dtype=od)
torch.cuda.synchronize()
print("ok")
