"""The one-shot P2P statistics exchange (include/cgbn.h cgbn_p2p_*; SURVEY 8(e) backend
2) on one GPU: cgbn_p2p_emulate runs the per-rank exchange routine as a cooperative
launch of G CTAs (CTA b = rank b, all co-resident, regions on the same device), so the
protocol -- push, epoch flags with release / acquire at system scope, double-buffered
receive area, rank-ordered output, timeout instead of a hang -- is checked without
separate kernels waiting on each other. The multi-process path (CUDA IPC regions,
DistHandle(transport="p2p")) runs the same device routine."""

import ctypes

import numpy as np
import pytest
import torch

from paper_1711_07240_b200 import _lib

pytestmark = pytest.mark.gpu


class Regions:
    def __init__(self, G, max_len):
        self.lib = _lib.load()
        nbytes = self.lib.cgbn_p2p_region_bytes(G, max_len)
        assert nbytes > 0
        self.ptrs = []
        for _ in range(G):
            p = ctypes.c_void_p()
            h = (ctypes.c_char * 64)()
            _lib.check(self.lib.cgbn_p2p_alloc(nbytes, ctypes.byref(p), h), "alloc")
            self.ptrs.append(p.value)
        self.arr, self.keep = _lib.ptr_array(self.ptrs)

    def free(self):
        torch.cuda.synchronize()
        for p in self.ptrs:
            self.lib.cgbn_p2p_free(p)


def _emulate(reg, vecs, max_len, timeout=5.0, skip=-1):
    lib = _lib.load()
    G, n = vecs.shape
    outs = torch.full((G, G * n), float("nan"), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(lib.cgbn_p2p_emulate(vecs.data_ptr(), n, G, reg.arr, max_len, outs.data_ptr(),
                                    status.data_ptr(), timeout, skip,
                                    torch.cuda.current_stream().cuda_stream), "emulate")
    torch.cuda.synchronize()
    return outs.view(G, G, n).cpu().numpy(), int(status.item())


@pytest.mark.parametrize("G,n", [(2, 129), (4, 2 * 256 + 1), (8, 4097), (8, 1)])
def test_p2p_protocol_many_epochs(G, n):
    """Every rank receives every rank's vector in rank order, epoch after epoch (both
    halves of the double buffer, varying lengths below max_len)."""
    max_len = 4097
    reg = Regions(G, max_len)
    rng = np.random.default_rng(G * 1000 + n)
    try:
        for it in range(6):
            m = max(1, n - it)  # lengths change between exchanges
            v = rng.standard_normal((G, m))
            outs, st = _emulate(reg, torch.from_numpy(v).cuda(), max_len)
            assert st == 0
            for b in range(G):
                assert np.array_equal(outs[b], v), (it, b)
    finally:
        reg.free()


def test_p2p_timeout_instead_of_hang():
    """A rank that never joins: the others give up after the timeout and flag it."""
    G, n, max_len = 4, 33, 64
    reg = Regions(G, max_len)
    try:
        v = torch.randn(G, n, dtype=torch.float64, device="cuda")
        outs, st = _emulate(reg, v, max_len, timeout=0.05, skip=2)
        assert st & _lib.STATUS_EXCHANGE_TIMEOUT
        for b in (0, 1, 3):  # the ranks that did arrive still exchanged among themselves
            for q in (0, 1, 3):
                assert np.array_equal(outs[b][q], v[q].cpu().numpy())
            assert np.isnan(outs[b][2]).all()  # the missing rank's row is NaN, not stale
    finally:
        reg.free()


def test_p2p_argument_validation():
    lib = _lib.load()
    assert lib.cgbn_p2p_region_bytes(0, 10) == 0
    assert lib.cgbn_p2p_region_bytes(4, 0) == 0
    v = torch.zeros(10, dtype=torch.float64, device="cuda")
    arr, keep = _lib.ptr_array([v.data_ptr()] * 2)
    rc = lib.cgbn_p2p_exchange(v.data_ptr(), 20, 0, 2, arr, 10, v.data_ptr(), None, 1.0, None)
    assert rc == _lib.ERR_INVALID
    assert b"outside" in lib.cgbn_last_error()


def _ipc_worker(rank, world, port, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1711_07240_b200 as cg
        h = cg.DistHandle(bn_group_size=world, transport="p2p", device="cuda:0",
                          p2p_max_len=1025)
        p = h._p2p
        res = {"rank": rank, "G": p.G, "idx": p.idx, "opened": len(p._opened),
               "regions": [p._keep[i] for i in range(p.G)]}
        h.close()
        dist.destroy_process_group()
        q.put(res)
    except Exception as exc:  # noqa: BLE001
        q.put({"rank": rank, "error": repr(exc)})


def test_p2p_ipc_setup_two_processes():
    """DistHandle(transport="p2p") host plumbing across two processes: allocate the
    region, share CUDA IPC handles, open the peer's region, close. No exchange kernel
    runs (two processes on one GPU must not wait on each other)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=180) for _ in range(2)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
    for d in out:
        assert "error" not in d, d
        assert d["G"] == 2 and d["opened"] == 1 and d["idx"] == d["rank"]
        assert all(r for r in d["regions"])


def test_p2p_exchange_kernel_in_cuda_graph_single_rank():
    """cgbn_p2p_exchange captured in a CUDA graph: the device-side epoch advances on every
    replay (both halves of the double buffer) and the fixed output follows the input.
    G = 1, so the kernel never waits on another rank."""
    lib = _lib.load()
    max_len, n = 64, 17
    reg = Regions(1, max_len)
    try:
        vec = torch.zeros(n, dtype=torch.float64, device="cuda")
        out = torch.zeros(n, dtype=torch.float64, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                _lib.check(lib.cgbn_p2p_exchange(vec.data_ptr(), n, 0, 1, reg.arr, max_len,
                                                 out.data_ptr(), status.data_ptr(), 1.0,
                                                 side.cuda_stream), "exchange")
        torch.cuda.current_stream().wait_stream(side)
        for it in range(5):
            vec.copy_(torch.arange(n, dtype=torch.float64, device="cuda") * (it + 1))
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, vec), it
        assert int(status.item()) == 0
    finally:
        reg.free()
