"""Producer fusion: the tcgen05 1x1 convolution whose epilogue emits
the BN forward partial (include/cgbn.h cgbn_conv1x1_stats, producer.py).

Checks, through the C ABI:
  * z against a float64 torch reference of the same bf16 operands. The tensor cores
    accumulate in fp32, so the error of an element is relative to the size of the
    products it sums, not to its own value: normwise max|z - ref| / max|ref| <= 1e-5 for
    fp32 z, plus one bf16 rounding (8e-3) for bf16 z;
  * the fused partial against the oracle's statistics of z *as stored* (f64): the
    epilogue accumulates the shifted sums of d = z - K in fp64 per element (d exact),
    so |mean error| <= 1e-12 std and the M2 relative error <= 1e-12, also with a channel
    offset of 1000 (|mean| >> std); for bf16 z the differences are summed in fp32 over
    groups of 8 first, as in the 16-bit BN statistics kernels (<= 2e-6);
  * the fused BN forward against the oracle on z (the reference's tolerances: 1e-5 on
    mean / var / y / running stats) for a single rank and a 4-rank group, and the
    backward through the resulting cache (1e-4 on dx / dgamma / dbeta);
  * tails: pixel tiles past H*W (3136 = 24.5 tiles), Cout below and not a multiple of
    128, Cin not a multiple of the 64-channel stage (TMA zero fill), bias, and a large
    channel mean (cancellation).
"""

import numpy as np
import pytest
import torch

from oracle import cgbn_oracle as O

import paper_1711_07240_b200 as cg
from paper_1711_07240_b200 import producer as P

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def _operands(n, cin, cout, hw, seed, loc=0.0, bias=False, bias_loc=0.0):
    g = torch.Generator().manual_seed(seed)
    h, w = hw
    x = (torch.randn(n, cin, h, w, generator=g) + loc).to(torch.bfloat16)
    wt = (torch.randn(cout, cin, generator=g) / cin ** 0.5).to(torch.bfloat16)
    b = torch.randn(cout, generator=g) * 3.0 + bias_loc if bias else None
    return x, wt, b


def _check_partial(p, mean, m2, cnt, cout, out_dtype=torch.float32):
    # fp32 z: fp64 per element (1e-12); bf16 z: fp32 sums over groups of 8 differences,
    # as the 16-bit BN statistics kernels do (<= 7 roundings of 2^-24 per group)
    tol = 1e-12 if out_dtype == torch.float32 else 2e-6
    assert p[2 * cout] == cnt
    std = np.sqrt(m2 / cnt)
    assert np.max(np.abs(p[:cout] - mean) / std) <= tol
    assert np.max(np.abs(p[cout:2 * cout] - m2) / m2) <= tol


def _z_ref(x, wt, b):
    z = torch.einsum("oc,nchw->nohw", wt.double(), x.double())
    if b is not None:
        z = z + b.double()[None, :, None, None]
    return z


def _stats64(z):
    a = z.double().cpu().numpy()
    c = a.shape[1]
    rows = a.transpose(1, 0, 2, 3).reshape(c, -1)
    mean = rows.mean(axis=1)
    m2 = ((rows - mean[:, None]) ** 2).sum(axis=1)
    return mean, m2, rows.shape[1]


SHAPES = [
    # n, cin, cout, (h, w)
    (2, 64, 256, (56, 56)),     # ResNet layer1 conv3 at batch 2, pixel tail of 64
    (3, 256, 64, (28, 28)),     # Cout below one 128-channel tile, 784 = 6.125 tiles
    (2, 72, 192, (10, 20)),     # Cin % 64 != 0 (K tail zero-filled), Cout % 128 != 0
    (1, 512, 128, (8, 8)),      # one pixel tile of 64 valid columns, 8 k-blocks
    (4, 128, 384, (16, 16)),    # exactly 2 pixel tiles per image
]


@pytest.mark.parametrize("n,cin,cout,hw", SHAPES)
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_conv_output_and_partial(n, cin, cout, hw, out_dtype):
    x, wt, b = _operands(n, cin, cout, hw, seed=cin + cout, bias=(cout % 128 != 0))
    _conv_case(x, wt, b, out_dtype)


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_partial_with_large_channel_offset(out_dtype):
    """bias 1000 +- 3: |mean| >> std (the cancellation case of the BN tests)."""
    x, wt, b = _operands(2, 64, 192, (28, 28), seed=7, bias=True, bias_loc=1000.0)
    _conv_case(x, wt, b, out_dtype)


def _conv_case(x, wt, b, out_dtype):
    n, _, h, w = x.shape
    cout = wt.shape[0]
    hw = (h, w)
    z, partial = P.conv1x1_stats(x.to(DEV), wt.to(DEV), b, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert z.dtype == out_dtype and z.shape == (n, cout, *hw)
    ref = _z_ref(x, wt, b)
    tol = 1e-5 if out_dtype == torch.float32 else 8e-3
    scale = float(ref.abs().max())
    assert O.rel_err(z.double().cpu().numpy(), ref.numpy(), floor=scale) <= tol
    mean, m2, cnt = _stats64(z)
    _check_partial(partial.cpu().numpy(), mean, m2, cnt, cout, out_dtype)
    # the plain conv writes the same z bitwise
    z2 = P.conv1x1(x.to(DEV), wt.to(DEV), b, out_dtype=out_dtype)
    assert torch.equal(z, z2)


def test_partial_matches_statistics_kernel():
    """The fused partial and cgbn_fwd_stats(z) describe the same statistics."""
    x, wt, _ = _operands(4, 64, 256, (56, 56), seed=5, loc=2.0)
    z, partial = P.conv1x1_stats(x.to(DEV), wt.to(DEV))
    lib = cg.batchnorm._lib.load()
    from paper_1711_07240_b200.tensor import stream_ptr, workspace
    c = 256
    hw = 56 * 56
    ws = workspace(DEV, lib.cgbn_workspace_bytes(4, c, hw, 0))
    p2 = torch.empty(2 * c + 1, dtype=torch.float64, device=DEV)
    cg.batchnorm._lib.check(lib.cgbn_fwd_stats(z.data_ptr(), 4, c, hw, 0, p2.data_ptr(),
                                               ws.data_ptr(), ws.numel(), stream_ptr(DEV)),
                            "cgbn_fwd_stats")
    _check_partial(partial.cpu().numpy(), p2[:c].cpu().numpy(), p2[c:2 * c].cpu().numpy(),
                   int(p2[-1]), c)


@pytest.mark.parametrize("bias_loc", [0.0, 1000.0])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_fused_bn_forward_local_matches_oracle(relu, out_dtype, bias_loc):
    n, cin, cout, hw = 2, 128, 256, (28, 28)
    x, wt, b = _operands(n, cin, cout, hw, seed=11, loc=1.0, bias=True, bias_loc=bias_loc)
    rng = np.random.default_rng(3)
    gamma = rng.uniform(0.5, 1.5, cout).astype(np.float32)
    beta = rng.standard_normal(cout).astype(np.float32)
    st = cg.BNLayerState(gamma=gamma, beta=beta)
    y, cache, z = P.conv1x1_bn_forward_local(x.to(DEV), wt.to(DEV), st, bias=b,
                                             out_dtype=out_dtype, relu=relu)
    dy = torch.randn(z.shape, generator=torch.Generator().manual_seed(4)).to(out_dtype)
    dx, dgamma, dbeta = cg.bn_backward_local(dy.to(DEV), cache, st)
    ref = O.cgbn_world([z.double().cpu().numpy()], gamma.astype(np.float64),
                       beta.astype(np.float64), 1, relu=relu,
                       dys=[dy.double().numpy()])[0]
    out_tol = 1e-5 if out_dtype == torch.float32 else 8e-3
    assert O.rel_err(cache.mu.cpu().numpy(), ref["mu"]) <= 1e-5
    assert O.rel_err(cache.var.cpu().numpy(), ref["var"]) <= 1e-5
    yref = torch.from_numpy(ref["y"]).to(out_dtype).double().numpy()
    assert O.rel_err(y.double().cpu().numpy(), yref) <= out_tol
    assert O.rel_err(st.running_mean.double().cpu().numpy(), ref["running_mean"]) <= 1e-5
    assert O.rel_err(st.running_var.double().cpu().numpy(), ref["running_var"]) <= 1e-5
    assert O.rel_err(dgamma.double().cpu().numpy(), ref["dgamma"]) <= 1e-4
    assert O.rel_err(dbeta.double().cpu().numpy(), ref["dbeta"]) <= 1e-4
    dx_tol = 1e-4 if out_dtype == torch.float32 else 8e-3
    dxref = torch.from_numpy(ref["dx"]).to(out_dtype).double().numpy()
    assert O.rel_err(dx.double().cpu().numpy(), dxref) <= dx_tol


def test_fused_equals_unfused_forward():
    """Same z, same BN state: the fused forward agrees with bn_forward_local(z)."""
    x, wt, _ = _operands(8, 256, 128, (14, 16), seed=21, loc=-3.0)
    st1 = cg.BNLayerState.create(128, device=DEV)
    st2 = cg.BNLayerState.create(128, device=DEV)
    y1, c1, z = P.conv1x1_bn_forward_local(x.to(DEV), wt.to(DEV), st1)
    y2, c2 = cg.bn_forward_local(z, st2)
    assert O.rel_err(y1.double().cpu().numpy(), y2.double().cpu().numpy()) <= 1e-5
    assert O.rel_err(c1.var.cpu().numpy(), c2.var.cpu().numpy()) <= 1e-12
    assert O.rel_err(st1.running_var.double().cpu().numpy(),
                     st2.running_var.double().cpu().numpy()) <= 1e-6


def test_sync_fused_forward_group_of_four():
    """4 ranks (one GPU, DeviceGroup), unequal batches: the group statistics of the fused
    path match the oracle on the concatenated z and are identical on every rank."""
    world, cin, cout, hw = 4, 64, 256, (28, 28)
    ops = [_operands(n, cin, cout, hw, seed=100 + r, loc=0.5) for r, n in enumerate([2, 1, 3, 2])]
    wt = ops[0][1]
    rng = np.random.default_rng(9)
    gamma = rng.uniform(0.5, 1.5, cout).astype(np.float32)
    beta = rng.standard_normal(cout).astype(np.float32)
    xs = [o[0].to(DEV) for o in ops]
    wd = wt.to(DEV)

    def worker(h):
        st = cg.BNLayerState(gamma=gamma, beta=beta)
        y, cache, z = P.sync_conv1x1_bn_forward(h, xs[h.rank], wd, st)
        return dict(y=y.double().cpu().numpy(), z=z.double().cpu().numpy(),
                    mu=cache.mu.cpu().numpy(), var=cache.var.cpu().numpy(),
                    rv=st.running_var.double().cpu().numpy())

    outs = cg.DeviceGroup(world, timeout_s=60.0).run(worker)
    ref = O.cgbn_world([o["z"] for o in outs], gamma.astype(np.float64),
                       beta.astype(np.float64), world)
    for r in range(world):
        assert np.array_equal(outs[r]["mu"], outs[0]["mu"])
        assert np.array_equal(outs[r]["var"], outs[0]["var"])
        assert O.rel_err(outs[r]["mu"], ref[r]["mu"]) <= 1e-5
        assert O.rel_err(outs[r]["var"], ref[r]["var"]) <= 1e-5
        assert O.rel_err(outs[r]["y"], ref[r]["y"]) <= 1e-5
        assert O.rel_err(outs[r]["rv"], ref[r]["running_var"]) <= 1e-5


def test_reference_exchange_mode_runs_unfused():
    prev = cg.set_forward_exchange("reference")
    try:
        x, wt, _ = _operands(2, 64, 128, (8, 8), seed=2)
        st = cg.BNLayerState.create(128, device=DEV)
        y, cache, z = P.conv1x1_bn_forward_local(x.to(DEV), wt.to(DEV), st)
        ref = O.cgbn_world([z.double().cpu().numpy()], np.ones(128), np.zeros(128), 1)[0]
        assert O.rel_err(y.double().cpu().numpy(), ref["y"]) <= 1e-5
    finally:
        cg.set_forward_exchange(prev)


def test_unsupported_shapes_raise():
    x = torch.randn(2, 64, 7, 7, device=DEV).to(torch.bfloat16)
    wt = torch.randn(128, 64, device=DEV).to(torch.bfloat16)
    with pytest.raises(cg.BatchNormError, match="multiples of 8"):
        P.conv1x1(x, wt)
    with pytest.raises(cg.BatchNormError, match="bfloat16"):
        P.conv1x1(x.float(), wt)


# ------------------------------------------- channels_last: 1x1 and 3x3 (TMA im2col)

def _cl(t):
    return t.contiguous(memory_format=torch.channels_last)


def _operands3(n, cin, cout, hw, seed, loc=0.0, bias=False, bias_loc=0.0):
    g = torch.Generator().manual_seed(seed)
    h, w = hw
    x = (torch.randn(n, cin, h, w, generator=g) + loc).to(torch.bfloat16)
    wt = (torch.randn(cout, cin, 3, 3, generator=g) / (9 * cin) ** 0.5).to(torch.bfloat16)
    b = torch.randn(cout, generator=g) * 3.0 + bias_loc if bias else None
    return x, wt, b


SHAPES_NHWC = [
    # n, cin, cout, (h, w): any H, W; tiles of 128 pixels run across rows and images
    (2, 64, 256, (56, 56)),
    (4, 256, 64, (14, 14)),     # H*W = 196: not possible on the NCHW kernel
    (3, 72, 136, (7, 7)),       # K tail, Cout % 128 != 0, 147 pixels
    (1, 512, 128, (5, 9)),
]


@pytest.mark.parametrize("n,cin,cout,hw", SHAPES_NHWC)
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_conv1x1_channels_last(n, cin, cout, hw, out_dtype):
    x, wt, b = _operands(n, cin, cout, hw, seed=cin * 3 + cout, bias=True)
    z, partial = P.conv1x1_stats(_cl(x.to(DEV)), wt.to(DEV), b, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert z.is_contiguous(memory_format=torch.channels_last) and z.shape == (n, cout, *hw)
    ref = _z_ref(x, wt, b)
    tol = 1e-5 if out_dtype == torch.float32 else 8e-3
    assert O.rel_err(z.double().cpu().numpy(), ref.numpy(), floor=float(ref.abs().max())) <= tol
    mean, m2, cnt = _stats64(z)
    _check_partial(partial.cpu().numpy(), mean, m2, cnt, cout, out_dtype)


SHAPES3 = [
    (2, 64, 64, (56, 56)),      # ResNet stage-1 conv2
    (2, 128, 128, (28, 28)),    # stage-2 conv2
    (3, 64, 256, (14, 14)),
    (1, 72, 192, (7, 7)),       # K tail, Cout tail, tiny plane (every pixel on a border)
    (2, 64, 64, (9, 13)),       # odd extents
]


def _z_ref3(x, wt, b):
    z = torch.nn.functional.conv2d(x.double(), wt.double(), padding=1)
    if b is not None:
        z = z + b.double()[None, :, None, None]
    return z


@pytest.mark.parametrize("n,cin,cout,hw", SHAPES3)
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_conv3x3_output_and_partial(n, cin, cout, hw, out_dtype):
    x, wt, b = _operands3(n, cin, cout, hw, seed=cin + cout + 3, bias=(cout % 128 != 0))
    z, partial = P.conv3x3_stats(_cl(x.to(DEV)), wt.to(DEV), b, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert z.is_contiguous(memory_format=torch.channels_last) and z.shape == (n, cout, *hw)
    ref = _z_ref3(x, wt, b)
    tol = 1e-5 if out_dtype == torch.float32 else 8e-3
    assert O.rel_err(z.double().cpu().numpy(), ref.numpy(), floor=float(ref.abs().max())) <= tol
    mean, m2, cnt = _stats64(z)
    _check_partial(partial.cpu().numpy(), mean, m2, cnt, cout, out_dtype)
    z2 = P.conv3x3(_cl(x.to(DEV)), wt.to(DEV), b, out_dtype=out_dtype)
    assert torch.equal(z, z2)


@pytest.mark.parametrize("bias_loc", [0.0, 1000.0])
def test_conv3x3_fused_bn_forward_backward_matches_oracle(bias_loc):
    n, cin, cout, hw = 2, 64, 128, (28, 28)
    x, wt, b = _operands3(n, cin, cout, hw, seed=31, loc=0.5, bias=True, bias_loc=bias_loc)
    rng = np.random.default_rng(5)
    gamma = rng.uniform(0.5, 1.5, cout).astype(np.float32)
    beta = rng.standard_normal(cout).astype(np.float32)
    st = cg.BNLayerState(gamma=gamma, beta=beta)
    y, cache, z = P.conv3x3_bn_forward_local(_cl(x.to(DEV)), wt.to(DEV), st, bias=b, relu=True)
    assert y.is_contiguous(memory_format=torch.channels_last)
    dy = torch.randn(z.shape, generator=torch.Generator().manual_seed(6))
    dx, dgamma, dbeta = cg.bn_backward_local(_cl(dy.to(DEV)), cache, st)
    ref = O.cgbn_world([z.double().cpu().numpy()], gamma.astype(np.float64),
                       beta.astype(np.float64), 1, relu=True, dys=[dy.double().numpy()])[0]
    yref = torch.from_numpy(ref["y"]).float().double().numpy()
    assert O.rel_err(y.double().cpu().numpy(), yref) <= 1e-5
    assert O.rel_err(cache.mu.cpu().numpy(), ref["mu"]) <= 1e-5
    assert O.rel_err(cache.var.cpu().numpy(), ref["var"]) <= 1e-5
    assert O.rel_err(st.running_mean.double().cpu().numpy(), ref["running_mean"]) <= 1e-5
    assert O.rel_err(st.running_var.double().cpu().numpy(), ref["running_var"]) <= 1e-5
    assert O.rel_err(dx.double().cpu().numpy(), ref["dx"]) <= 1e-4
    assert O.rel_err(dgamma.double().cpu().numpy(), ref["dgamma"]) <= 1e-4
    assert O.rel_err(dbeta.double().cpu().numpy(), ref["dbeta"]) <= 1e-4


def test_sync_conv3x3_group_of_two():
    """Two ranks with unequal batches: group statistics identical on both ranks and equal
    to the oracle on the concatenated z."""
    world, cin, cout, hw = 2, 64, 64, (14, 14)
    ops = [_operands3(n, cin, cout, hw, seed=200 + r) for r, n in enumerate([2, 3])]
    wd = ops[0][1].to(DEV)
    xs = [_cl(o[0].to(DEV)) for o in ops]

    def worker(h):
        st = cg.BNLayerState.create(cout, device=DEV)
        y, cache, z = P.sync_conv3x3_bn_forward(h, xs[h.rank], wd, st)
        return dict(y=y.double().cpu().numpy(), z=z.double().cpu().numpy(),
                    mu=cache.mu.cpu().numpy(), var=cache.var.cpu().numpy())

    outs = cg.DeviceGroup(world, timeout_s=60.0).run(worker)
    ref = O.cgbn_world([o["z"] for o in outs], np.ones(cout), np.zeros(cout), world)
    for r in range(world):
        assert np.array_equal(outs[r]["var"], outs[0]["var"])
        assert O.rel_err(outs[r]["var"], ref[r]["var"]) <= 1e-5
        assert O.rel_err(outs[r]["y"], ref[r]["y"]) <= 1e-5


def test_conv3x3_needs_channels_last():
    x = torch.randn(1, 64, 8, 8, device=DEV).to(torch.bfloat16)
    wt = torch.randn(64, 64, 3, 3, device=DEV).to(torch.bfloat16)
    with pytest.raises(cg.BatchNormError, match="channels_last"):
        P.conv3x3(x, wt)


STRIDED = [
    # k, n, cin, cout, (h, w): stride 2 (ResNet's first-block conv2 and 1x1 downsample)
    (3, 2, 64, 128, (56, 56)),
    (3, 3, 128, 64, (15, 9)),    # odd extents: Ho = 8, Wo = 5
    (1, 2, 256, 512, (56, 56)),  # the 1x1 downsample
    (1, 1, 64, 72, (7, 13)),
]


@pytest.mark.parametrize("k,n,cin,cout,hw", STRIDED)
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_strided_conv_channels_last(k, n, cin, cout, hw, out_dtype):
    if k == 3:
        x, wt, b = _operands3(n, cin, cout, hw, seed=k + cin + cout, bias=True)
        z, partial = P.conv3x3_stats(_cl(x.to(DEV)), wt.to(DEV), b, out_dtype=out_dtype,
                                     stride=2)
    else:
        x, wt, b = _operands(n, cin, cout, hw, seed=k + cin + cout, bias=True)
        z, partial = P.conv1x1_stats(_cl(x.to(DEV)), wt.to(DEV), b, out_dtype=out_dtype,
                                     stride=2)
    torch.cuda.synchronize()
    w4 = wt.double() if k == 3 else wt.double()[:, :, None, None]
    ref = torch.nn.functional.conv2d(x.double(), w4, stride=2, padding=k // 2)
    ref = ref + b.double()[None, :, None, None]
    assert z.shape == ref.shape and z.is_contiguous(memory_format=torch.channels_last)
    tol = 1e-5 if out_dtype == torch.float32 else 8e-3
    assert O.rel_err(z.double().cpu().numpy(), ref.numpy(), floor=float(ref.abs().max())) <= tol
    mean, m2, cnt = _stats64(z)
    _check_partial(partial.cpu().numpy(), mean, m2, cnt, cout, out_dtype)


def test_strided_fused_bn_forward_matches_oracle():
    x, wt, b = _operands3(4, 64, 128, (28, 28), seed=77, loc=0.3, bias=True)
    st = cg.BNLayerState.create(128, device=DEV)
    y, cache, z = P.conv3x3_bn_forward_local(_cl(x.to(DEV)), wt.to(DEV), st, bias=b, stride=2)
    assert z.shape == (4, 128, 14, 14)
    ref = O.cgbn_world([z.double().cpu().numpy()], np.ones(128), np.zeros(128), 1)[0]
    assert O.rel_err(y.double().cpu().numpy(), ref["y"]) <= 1e-5
    assert O.rel_err(cache.var.cpu().numpy(), ref["var"]) <= 1e-5


def test_strided_nchw_raises():
    x = torch.randn(2, 64, 8, 8, device=DEV).to(torch.bfloat16)
    wt = torch.randn(64, 64, device=DEV).to(torch.bfloat16)
    with pytest.raises(cg.BatchNormError, match="channels_last"):
        P.conv1x1(x, wt, stride=2)
