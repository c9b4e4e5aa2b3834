"""Debug helper: fused conv partial vs f64 statistics of z, per channel."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_07240_b200 import producer as P
dev = torch.device("cuda", 0)
for (n, cin, cout, h, w, bl) in [(2, 128, 256, 28, 28, 1000.0), (2, 128, 256, 28, 28, 0.0), (1, 512, 128, 8, 8, 0.0)]:
    g = torch.Generator().manual_seed(11)
    x = (torch.randn(n, cin, h, w, generator=g) + 1.0).to(torch.bfloat16)
    wt = (torch.randn(cout, cin, generator=g) / cin ** 0.5).to(torch.bfloat16)
    b = torch.randn(cout, generator=g) * 3.0 + bl
    z, p = P.conv1x1_stats(x.to(dev), wt.to(dev), b)
    torch.cuda.synchronize()
    a = z.double().cpu().numpy().transpose(1, 0, 2, 3).reshape(cout, -1)
    mean = a.mean(1); m2 = ((a - mean[:, None]) ** 2).sum(1); std = np.sqrt(m2 / a.shape[1])
    p = p.cpu().numpy()
    em = np.abs(p[:cout] - mean) / std; e2 = np.abs(p[cout:2*cout] - m2) / m2
    print((n, cin, cout, h, w, bl), "count", p[-1], a.shape[1], "mean err/std max %.3g" % em.max(), "ch", em.argmax(),
          "M2 rel err max %.3g" % e2.max(), "ch", e2.argmax(), "std range", std.min(), std.max())

# BN on z at a 1000 offset: fused partial vs the split path vs the oracle
import paper_1711_07240_b200 as cg
from oracle import cgbn_oracle as O
g = torch.Generator().manual_seed(11)
n, cin, cout, h, w = 2, 128, 256, 28, 28
x = (torch.randn(n, cin, h, w, generator=g) + 1.0).to(torch.bfloat16)
wt = (torch.randn(cout, cin, generator=g) / cin ** 0.5).to(torch.bfloat16)
b = torch.randn(cout, generator=g) * 3.0 + 1000.0
rng = np.random.default_rng(3)
gamma = rng.uniform(0.5, 1.5, cout).astype(np.float32)
beta = rng.standard_normal(cout).astype(np.float32)
st1 = cg.BNLayerState(gamma=gamma, beta=beta)
y1, c1, z = P.conv1x1_bn_forward_local(x.to(dev), wt.to(dev), st1, bias=b)
st2 = cg.BNLayerState(gamma=gamma, beta=beta)
y2, c2 = cg.bn_forward_local(z, st2)
ref = O.cgbn_world([z.double().cpu().numpy()], gamma.astype(np.float64), beta.astype(np.float64), 1)[0]
yr = torch.from_numpy(ref["y"]).float().double().numpy()
for name, y, c in (("fused", y1, c1), ("split", y2, c2)):
    yy = y.double().cpu().numpy()
    err = np.abs(yy - yr) / np.maximum(np.maximum(np.abs(yy), np.abs(yr)), 1e-3)
    i = np.unravel_index(err.argmax(), err.shape)
    print(name, "y rel_err %.3g" % err.max(), "at", i, "y", yy[i], "ref", yr[i], "ref64", ref["y"][i],
          "mu err %.3g" % np.abs(c.mu.cpu().numpy() - ref["mu"]).max(),
          "var rel %.3g" % (np.abs(c.var.cpu().numpy() - ref["var"]) / ref["var"]).max())
