"""The NCCL statistics exchange inside a CUDA graph (bench.py captures the whole step,
exchanges included, when it runs one process per GPU under torchrun; SURVEY 8(e)
backend 1).

A single GPU cannot host two NCCL ranks, so this runs a one-rank NCCL job in a
subprocess: the all-gather of `DistHandle.exchange` (`_all_gather_rows`) and the sharded
allreduce (all-to-all + all-gather) are captured in a CUDA graph after a warm-up call,
replayed with new inputs, and must reproduce the eager results bitwise. It also captures
a DistHandle BN forward + backward step the way bench.py does."""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import torch, torch.distributed as dist
import paper_1711_07240_b200 as cg
from paper_1711_07240_b200 import collectives as co

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
h = cg.DistHandle(bn_group_size=1)

# 1) the exchange collectives captured in a graph
v = torch.randn(2 * 256 + 1, device=dev, dtype=torch.float64)
big = torch.randn(co.SHARDED_MIN_ELEMS + 3, device=dev, dtype=torch.float64)
s = torch.cuda.Stream(device=dev)
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    co._all_gather_rows(v, 1, None)            # communicator warm-up before capture
    co._sharded_allreduce(big, 1, None, co._device_fold)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    out = co._all_gather_rows(v, 1, None)
    red = co._sharded_allreduce(big, 1, None, co._device_fold)
for it in range(3):
    v.copy_(torch.randn_like(v))
    big.copy_(torch.randn_like(big))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out[0], v), "captured all-gather differs"
    assert torch.equal(red, big), "captured sharded allreduce differs"

# 2) a BN forward + backward step on a DistHandle, captured like bench.py's step
shapes = [(4, 64, 14, 14), (4, 256, 7, 7)]
gen = torch.Generator(device=dev); gen.manual_seed(0)
xs = [torch.randn(sh, device=dev, generator=gen) for sh in shapes]
dys = [torch.randn(sh, device=dev, generator=gen) for sh in shapes]
sts = [cg.BNLayerState(gamma=torch.rand(sh[1], device=dev) + 0.5,
                       beta=torch.randn(sh[1], device=dev)) for sh in shapes]
res = {}
def step():
    caches = []
    for i, (x, st) in enumerate(zip(xs, sts)):
        y, c = cg.sync_bn_forward(h, x, st)
        res[("y", i)] = y
        caches.append(c)
    for i in range(len(xs) - 1, -1, -1):
        dx, dg, db = cg.sync_bn_backward(h, dys[i], caches[i], sts[i])
        res[("dx", i)] = dx
with torch.cuda.stream(s):
    step()
torch.cuda.synchronize()
eager = {k: t.clone() for k, t in res.items()}
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    step()
g2.replay()
torch.cuda.synchronize()
for k, t in eager.items():
    assert torch.equal(res[k], t), f"captured BN step differs at {k}"
dist.destroy_process_group()
print("nccl graph ok")
"""


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_nccl_exchange_and_bn_step_capture_in_cuda_graph():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()),
               RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "nccl graph ok" in r.stdout
