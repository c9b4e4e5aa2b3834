"""Debug helper: fused conv partial vs f64 statistics of z, per channel."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_07240_b200 import producer as P
dev = torch.device("cuda", 0)
for (n, cin, cout, h, w) in [(1, 64, 128, 8, 16), (1, 64, 128, 16, 16), (2, 64, 128, 8, 16), (1, 64, 128, 8, 8)]:
    g = torch.Generator().manual_seed(0)
    x = torch.randn(n, cin, h, w, generator=g).to(torch.bfloat16)
    wt = (torch.randn(cout, cin, generator=g) / 8).to(torch.bfloat16)
    z, p = P.conv1x1_stats(x.to(dev), wt.to(dev))
    torch.cuda.synchronize()
    a = z.double().cpu().numpy().transpose(1, 0, 2, 3).reshape(cout, -1)
    mean = a.mean(1); m2 = ((a - mean[:, None]) ** 2).sum(1)
    p = p.cpu().numpy()
    em = np.abs(p[:cout] - mean); e2 = np.abs(p[cout:2*cout] - m2) / m2
    print((n, cin, cout, h, w), "count", p[-1], a.shape[1], "mean abs err max", em.max(), "argmax", em.argmax(),
          "M2 rel err max", e2.max(), "argmax", e2.argmax())
    c = int(em.argmax())
    print("   ch", c, "gpu", p[c], p[cout + c], "ref", mean[c], m2[c], "sum ref", a[c].sum())
