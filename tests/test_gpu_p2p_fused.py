"""The P2P exchange fused into the kernels on either side of it (include/cgbn.h
cgbn_*_p2p; SURVEY 8(e) backend 3): the statistics reduction's channel finishers push the
rank's partial into every rank's region and the last one publishes; the finalize kernel
waits for the flags and folds the rows in place.

On one GPU (regions all local, as in test_gpu_p2p.py) the G ranks run one after another:
every rank's reduction (push + publish) first, then every rank's consumer, whose flags
are already set — no kernel ever waits on another one that is running. The results must
equal the unfused path (cgbn_fwd_stats / cgbn_bwd_reduce, gathered partials,
cgbn_fwd_normalize / cgbn_bwd_dx) bitwise, epoch after epoch (both buffer halves), for
the reduction families the planner picks (NCHW cluster-team and flat, channels_last rows,
2-D), and a rank that never publishes must produce the timeout status, not a hang.
"""

import ctypes

import numpy as np
import pytest
import torch

from paper_1711_07240_b200 import _lib
from paper_1711_07240_b200.tensor import stream_ptr

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)
MAX_LEN = 2 * 2048 + 1


class Regions:
    def __init__(self, G):
        self.lib = _lib.load()
        nbytes = self.lib.cgbn_p2p_region_bytes(G, MAX_LEN)
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


def _layout(x):
    lay = _lib.LAYOUT_NHWC if (x.dim() == 4 and x.is_contiguous(memory_format=torch.channels_last)
                               and not x.is_contiguous()) else _lib.LAYOUT_NCHW
    n, c = x.shape[:2]
    hw = x.numel() // (n * c)
    act = {torch.float32: _lib.ACT_F32, torch.bfloat16: _lib.ACT_BF16,
           torch.float16: _lib.ACT_F16}[x.dtype]
    return n, c, hw, lay | act


class Rank:
    def __init__(self, x, dy, gamma, beta):
        self.x, self.dy = x, dy
        self.n, self.c, self.hw, self.lay = _layout(x)
        self.gamma, self.beta = gamma, beta
        lib = _lib.load()
        self.ws = torch.zeros(lib.cgbn_workspace_bytes(self.n, self.c, self.hw, self.lay),
                              dtype=torch.uint8, device=DEV)
        self.status = torch.zeros(1, dtype=torch.int32, device=DEV)
        self.rm = torch.zeros(self.c, device=DEV)
        self.rv = torch.ones(self.c, device=DEV)

    def outputs(self):
        c = self.c
        self.y = torch.empty_like(self.x)
        self.dx = torch.empty_like(self.x)
        self.saved = torch.empty(3 * c + 1, dtype=torch.float64, device=DEV)
        self.dg = torch.empty(c, device=DEV)
        self.db = torch.empty(c, device=DEV)


def _fused_step(lib, ranks, reg, st, relu, skip=-1, timeout=5.0):
    G = len(ranks)
    for r, k in enumerate(ranks):
        k.outputs()
        if r == skip:
            continue
        _lib.check(lib.cgbn_fwd_stats_p2p(k.x.data_ptr(), k.n, k.c, k.hw, k.lay, r, G, reg.arr,
                                          MAX_LEN, k.ws.data_ptr(), k.ws.numel(), st),
                   "cgbn_fwd_stats_p2p")
    for r, k in enumerate(ranks):
        if r == skip:
            continue
        _lib.check(lib.cgbn_fwd_normalize_p2p(
            k.x.data_ptr(), k.n, k.c, k.hw, k.lay, reg.ptrs[r], G, MAX_LEN, timeout,
            k.gamma.data_ptr(), k.beta.data_ptr(), 1e-5, 0.1, k.rm.data_ptr(), k.rv.data_ptr(),
            k.saved.data_ptr(), int(relu), k.y.data_ptr(), k.status.data_ptr(), k.ws.data_ptr(),
            k.ws.numel(), st), "cgbn_fwd_normalize_p2p")
    if skip >= 0:
        return
    for r, k in enumerate(ranks):
        _lib.check(lib.cgbn_bwd_reduce_p2p(
            k.dy.data_ptr(), k.x.data_ptr(), k.n, k.c, k.hw, k.lay, k.saved.data_ptr(),
            k.gamma.data_ptr(), k.beta.data_ptr(), int(relu), r, G, reg.arr, MAX_LEN,
            k.ws.data_ptr(), k.ws.numel(), st), "cgbn_bwd_reduce_p2p")
    for r, k in enumerate(ranks):
        _lib.check(lib.cgbn_bwd_dx_p2p(
            k.dy.data_ptr(), k.x.data_ptr(), k.n, k.c, k.hw, k.lay, reg.ptrs[r], G, MAX_LEN,
            timeout, k.saved.data_ptr(), k.gamma.data_ptr(), k.beta.data_ptr(), 1e-5, int(relu),
            k.dx.data_ptr(), k.dg.data_ptr(), k.db.data_ptr(), k.status.data_ptr(),
            k.ws.data_ptr(), k.ws.numel(), st), "cgbn_bwd_dx_p2p")


def _split_step(lib, ranks, st, relu):
    """The unfused path on the same inputs: partials gathered in rank order."""
    G = len(ranks)
    parts = []
    for k in ranks:
        k.outputs()
        p = torch.empty(2 * k.c + 1, dtype=torch.float64, device=DEV)
        _lib.check(lib.cgbn_fwd_stats(k.x.data_ptr(), k.n, k.c, k.hw, k.lay, p.data_ptr(),
                                      k.ws.data_ptr(), k.ws.numel(), st), "cgbn_fwd_stats")
        parts.append(p)
    arr, keep = _lib.ptr_array([p.data_ptr() for p in parts])
    for k in ranks:
        _lib.check(lib.cgbn_fwd_normalize(
            k.x.data_ptr(), k.n, k.c, k.hw, k.lay, arr, G, k.gamma.data_ptr(), k.beta.data_ptr(),
            1e-5, 0.1, k.rm.data_ptr(), k.rv.data_ptr(), k.saved.data_ptr(), int(relu),
            k.y.data_ptr(), k.status.data_ptr(), k.ws.data_ptr(), k.ws.numel(), st),
            "cgbn_fwd_normalize")
    bparts = []
    for k in ranks:
        p = torch.empty(2 * k.c, dtype=torch.float64, device=DEV)
        _lib.check(lib.cgbn_bwd_reduce(
            k.dy.data_ptr(), k.x.data_ptr(), k.n, k.c, k.hw, k.lay, k.saved.data_ptr(),
            k.gamma.data_ptr(), k.beta.data_ptr(), int(relu), p.data_ptr(), k.ws.data_ptr(),
            k.ws.numel(), st), "cgbn_bwd_reduce")
        bparts.append(p)
    barr, bkeep = _lib.ptr_array([p.data_ptr() for p in bparts])
    for k in ranks:
        _lib.check(lib.cgbn_bwd_dx(
            k.dy.data_ptr(), k.x.data_ptr(), k.n, k.c, k.hw, k.lay, barr, G, k.saved.data_ptr(),
            k.gamma.data_ptr(), k.beta.data_ptr(), 1e-5, int(relu), k.dx.data_ptr(),
            k.dg.data_ptr(), k.db.data_ptr(), k.status.data_ptr(), k.ws.data_ptr(), k.ws.numel(),
            st), "cgbn_bwd_dx")
    torch.cuda.synchronize()


def _make_ranks(G, shape, seed, channels_last=False, dtype=torch.float32):
    g = torch.Generator().manual_seed(seed)
    c = shape[1]
    gamma = (torch.rand(c, generator=g) + 0.5).to(DEV)
    beta = torch.randn(c, generator=g).to(DEV)
    ranks = []
    for r in range(G):
        s = (shape[0] + r % 2,) + tuple(shape[1:])  # unequal batches
        x = (torch.randn(s, generator=g) + 1.0).to(DEV).to(dtype)
        dy = torch.randn(s, generator=g).to(DEV).to(dtype)
        if channels_last:
            x = x.contiguous(memory_format=torch.channels_last)
            dy = dy.contiguous(memory_format=torch.channels_last)
        ranks.append(Rank(x, dy, gamma, beta))
    return ranks


CASES = [
    # G, per-rank shape, channels_last, dtype
    (2, (8, 256, 28, 28), False, torch.float32),     # cluster-team reduction
    (4, (2, 64, 14, 14), False, torch.float32),      # small C
    (8, (1, 2048, 7, 7), False, torch.float32),      # SURVEY config 5 (latency-bound)
    (4, (4, 128, 14, 14), True, torch.float32),      # channels_last rows reduction
    (2, (64, 512), False, torch.float32),            # 2-D (N, C)
    (4, (4, 96, 12, 12), True, torch.bfloat16),
]


@pytest.mark.parametrize("G,shape,cl,dtype", CASES)
@pytest.mark.parametrize("relu", [False, True])
def test_fused_exchange_equals_split_path(G, shape, cl, dtype, relu):
    lib = _lib.load()
    st = stream_ptr(DEV)
    reg = Regions(G)
    try:
        fused = _make_ranks(G, shape, seed=G * 7 + shape[1], channels_last=cl, dtype=dtype)
        split = _make_ranks(G, shape, seed=G * 7 + shape[1], channels_last=cl, dtype=dtype)
        for epoch in range(3):  # both halves of the double buffer, running stats advance
            _fused_step(lib, fused, reg, st, relu)
            _split_step(lib, split, st, relu)
            for a, b in zip(fused, split):
                assert int(a.status.item()) == 0
                for name in ("y", "dx", "saved", "dg", "db", "rm", "rv"):
                    assert torch.equal(getattr(a, name), getattr(b, name)), (epoch, name)
    finally:
        reg.free()


def test_fused_exchange_missing_rank_times_out():
    lib = _lib.load()
    st = stream_ptr(DEV)
    G = 4
    reg = Regions(G)
    try:
        ranks = _make_ranks(G, (2, 64, 8, 8), seed=3)
        _fused_step(lib, ranks, reg, st, relu=False, skip=2, timeout=0.05)
        torch.cuda.synchronize()
        for r, k in enumerate(ranks):
            if r != 2:
                assert int(k.status.item()) & _lib.STATUS_EXCHANGE_TIMEOUT
                # the missing rank's stale rows are never folded: the layer state is left
                # as it was and the outputs are NaN (no silent stale statistics)
                assert torch.equal(k.rm, torch.zeros_like(k.rm))
                assert torch.equal(k.rv, torch.ones_like(k.rv))
                assert bool(torch.isnan(k.y).all())
    finally:
        reg.free()


def test_fused_exchange_rejects_large_groups():
    lib = _lib.load()
    x = torch.randn(2, 8, 4, 4, device=DEV)
    ws = torch.zeros(lib.cgbn_workspace_bytes(2, 8, 16, 0), dtype=torch.uint8, device=DEV)
    arr, keep = _lib.ptr_array([x.data_ptr()] * 9)
    rc = lib.cgbn_fwd_stats_p2p(x.data_ptr(), 2, 8, 16, 0, 0, 9, arr, MAX_LEN, ws.data_ptr(),
                                ws.numel(), stream_ptr(DEV))
    assert rc == _lib.ERR_INVALID and b"group size" in lib.cgbn_last_error()


def test_fused_exchange_replays_in_a_cuda_graph():
    """The epoch lives on the device: a captured fused step (every rank's reductions, then
    every rank's consumers) replayed several times keeps matching the split path."""
    lib = _lib.load()
    G = 4
    reg = Regions(G)
    try:
        fused = _make_ranks(G, (2, 128, 14, 14), seed=5)
        split = _make_ranks(G, (2, 128, 14, 14), seed=5)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for k in fused:
                k.outputs()  # allocate the outputs before capture
            _fused_step(lib, fused, reg, s.cuda_stream, relu=True)  # warm-up epoch
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            keep = [(k.y, k.dx, k.saved, k.dg, k.db) for k in fused]

            def no_alloc_outputs(self=None):
                pass
            orig = Rank.outputs
            Rank.outputs = no_alloc_outputs  # the graph writes the buffers captured above
            try:
                with torch.cuda.graph(g, stream=s):
                    _fused_step(lib, fused, reg, s.cuda_stream, relu=True)
            finally:
                Rank.outputs = orig
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
        st = stream_ptr(DEV)
        for _ in range(1 + 3):  # warm-up epoch + 3 replays (the capture itself runs nothing)
            _split_step(lib, split, st, relu=True)
        for a, b in zip(fused, split):
            assert int(a.status.item()) == 0
            for name in ("y", "dx", "saved", "dg", "db", "rm", "rv"):
                assert torch.equal(getattr(a, name), getattr(b, name)), name
        del keep
    finally:
        reg.free()
