"""The single-launch on-chip passes (csrc/cgbn_onchip.cuh) against the oracle, forced
through cgbn_fwd_fused / cgbn_bwd_fused (set_fused) on shapes that exercise every
branch: aligned planes (16-byte chunks) and odd planes (masked covers, two-channel write
chunks), one and several channels per cluster, clusters of 1..8 CTAs, ReLU, shifted
means, fp32 / bf16 / fp16; plus the statistics-only mode that multi-rank groups use for
on-chip-selected layers (bitwise the local statistics for identical shards,
test_batchnorm.py:252-262).

Tolerances: tests/test_gpu_parity.py (fp32), tests/test_gpu_half.py (16-bit outputs)."""

import numpy as np
import pytest
import torch

from oracle import cgbn_oracle as O

import paper_1711_07240_b200 as cg
from paper_1711_07240_b200 import _lib

pytestmark = pytest.mark.gpu

OUT_TOL = {torch.float32: (1e-5, 1e-4), torch.bfloat16: (8e-3, 8e-3),
           torch.float16: (1.5e-3, 1.5e-3)}


def _case(shape, seed, loc, dtype, relu):
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(seed)
    c = shape[1]
    x = (loc + rng.standard_normal(shape)).astype(np.float32)
    dy = rng.standard_normal(shape).astype(np.float32)
    xt = torch.from_numpy(x).to(dev).to(dtype)
    dyt = torch.from_numpy(dy).to(dev).to(dtype)
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.standard_normal(c).astype(np.float32)
    st = cg.BNLayerState(gamma=gamma, beta=beta)
    y, cache = cg.bn_forward_local(xt, st, relu=relu)
    dx, dg, db = cg.bn_backward_local(dyt, cache, st)
    ref = O.cgbn_world([xt.double().cpu().numpy()], gamma.astype(np.float64),
                       beta.astype(np.float64), 1, relu=relu,
                       dys=[dyt.double().cpu().numpy()])[0]
    return y, cache, dx, dg, db, st, ref


@pytest.mark.parametrize("shape,loc,relu", [
    ((32, 128, 28, 28), 0.0, False),   # aligned, one channel per cluster, KC > 1
    ((32, 256, 14, 14), 3.0, True),    # aligned 14x14, ReLU, shifted mean
    ((8, 64, 7, 7), 0.0, True),        # odd planes, several channels per CTA
    ((4, 256, 13, 21), 1000.0, False),  # odd 273-element planes, adversarial mean
    ((4, 20, 9, 9), 0.0, False),       # C not a power of two: a partial last cluster
    ((1, 2048, 7, 7), 0.0, False),     # config 5 layer: one image
])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
def test_forced_onchip_matches_oracle(shape, loc, relu, dtype):
    lib = _lib.load()
    act = {torch.float32: 0, torch.bfloat16: _lib.ACT_BF16, torch.float16: _lib.ACT_F16}[dtype]
    n, c, h, w = shape
    assert lib.cgbn_fused_supported(n, c, h * w, act, 0) == 1
    prev = cg.set_fused(True)
    try:
        y, cache, dx, dg, db, st, ref = _case(shape, sum(shape), loc, dtype, relu)
    finally:
        cg.set_fused(prev)
    ty, tdx = OUT_TOL[dtype]
    want_y = torch.from_numpy(ref["y"]).to(dtype).double().numpy() if dtype != torch.float32 \
        else ref["y"]
    assert O.rel_err(y.double().cpu().numpy(), want_y) <= ty
    assert O.rel_err(cache.mu.cpu().numpy(), ref["mu"]) <= 1e-5
    assert O.rel_err(cache.var.cpu().numpy(), ref["var"]) <= 1e-5
    assert O.rel_err(st.running_mean.cpu().numpy(), ref["running_mean"]) <= 1e-5
    assert O.rel_err(st.running_var.cpu().numpy(), ref["running_var"]) <= 1e-5
    assert O.rel_err(dg.cpu().numpy(), ref["dgamma"]) <= 1e-4
    assert O.rel_err(db.cpu().numpy(), ref["dbeta"]) <= 1e-4
    want_dx = torch.from_numpy(ref["dx"]).to(dtype).double().numpy() if dtype != torch.float32 \
        else ref["dx"]
    assert O.rel_err(dx.double().cpu().numpy(), want_dx) <= tdx


@pytest.mark.parametrize("shape", [(32, 128, 28, 28), (4, 96, 7, 7), (32, 256, 14, 14)])
def test_statistics_only_mode_bitwise_local(shape):
    """Identical shards on a 2-rank group: the group statistics equal the local ones
    bitwise (test_batchnorm.py:252-262) also when the layer runs on chip -- the group's
    partials come from the same on-chip reduction, in its statistics-only mode."""
    lib = _lib.load()
    n, c, h, w = shape
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(np.random.default_rng(8).standard_normal(shape).astype(np.float32)).to(dev)
    dy = torch.from_numpy(np.random.default_rng(9).standard_normal(shape).astype(np.float32)).to(dev)
    gamma = np.random.default_rng(10).uniform(0.5, 1.5, c).astype(np.float32)
    beta = np.zeros(c, np.float32)

    def worker(hd):
        st = cg.BNLayerState(gamma=gamma, beta=beta)
        y, cache = cg.sync_bn_forward(hd, x, st)
        dxg, dgg, dbg = cg.sync_bn_backward(hd, dy, cache, st)
        return cache.mu.cpu().numpy(), cache.var.cpu().numpy(), dgg.cpu().numpy() / 2

    out = cg.DeviceGroup(2).run(worker)
    st = cg.BNLayerState(gamma=gamma, beta=beta)
    _, cache = cg.bn_forward_local(x, st)
    _, dg, _ = cg.bn_backward_local(dy, cache, st)
    for r in range(2):
        assert np.array_equal(out[r][0], cache.mu.cpu().numpy())
        assert np.array_equal(out[r][1], cache.var.cpu().numpy())
        # group dgamma = 2 x the local one, exactly (sums of two identical fp64 partials)
        assert np.array_equal(out[r][2], dg.cpu().numpy())
    assert lib.cgbn_onchip_selected(n, c, h * w, 0, 0) == 1
