"""bf16 / fp16 activations: storage only -- every statistic is fp64,
gamma / beta / running statistics stay fp32, outputs are rounded once to the activation
dtype. The oracle runs in f64 on the same rounded inputs.

Tolerances (rel_err with the reference's 1e-3 floor, pkg/tests/helpers.py:158-163):
    mean, var, running_mean, running_var          1e-5  (fp64 sums of exact inputs)
    dgamma, dbeta (fp32 outputs)                  1e-4
    y, x_hat, dx in bf16: 8e-3 (one rounding, 2^-8 relative); in fp16: 1.5e-3 (2^-11,
    plus the 1e-3 floor applied to values just above fp16's subnormal range)
"""

import numpy as np
import pytest
import torch

from oracle import cgbn_oracle as O

import paper_1711_07240_b200 as cg

pytestmark = pytest.mark.gpu

OUT_TOL = {torch.bfloat16: 8e-3, torch.float16: 1.5e-3}


def _case(shapes, dtype, seed, loc=0.0, relu=False):
    rng = np.random.default_rng(seed)
    c = shapes[0][1]
    xs = [torch.from_numpy((loc + rng.standard_normal(s)).astype(np.float32)).to(dtype)
          for s in shapes]
    dys = [torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(dtype) for s in shapes]
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.standard_normal(c).astype(np.float32)
    ref = O.cgbn_world([x.double().numpy() for x in xs], gamma.astype(np.float64),
                       beta.astype(np.float64), len(shapes), relu=relu,
                       dys=[d.double().numpy() for d in dys])
    return xs, dys, gamma, beta, ref


def _run(xs, dys, gamma, beta, relu=False, channels_last=False):
    dev = torch.device("cuda", 0)
    xs = [x.to(dev) for x in xs]
    dys = [d.to(dev) for d in dys]
    if channels_last:
        xs = [x.contiguous(memory_format=torch.channels_last) for x in xs]
        dys = [d.contiguous(memory_format=torch.channels_last) for d in dys]

    def worker(h):
        st = cg.BNLayerState(gamma=gamma, beta=beta)
        y, cache = cg.sync_bn_forward(h, xs[h.rank], st, relu=relu)
        dx, dgamma, dbeta = cg.sync_bn_backward(h, dys[h.rank], cache, st)
        assert y.dtype == xs[h.rank].dtype and dx.dtype == xs[h.rank].dtype
        assert dgamma.dtype == torch.float32
        if channels_last:
            assert y.is_contiguous(memory_format=torch.channels_last)
        out = dict(y=y, x_hat=cache.x_hat, dx=dx, mu=cache.mu, var=cache.var, dgamma=dgamma,
                   dbeta=dbeta, running_mean=st.running_mean, running_var=st.running_var)
        return {k: v.detach().double().cpu().numpy() for k, v in out.items()}

    return cg.DeviceGroup(len(xs), timeout_s=60.0).run(worker)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("shapes,relu,loc,cl", [
    ([(2, 64, 56, 56)] * 2, False, 0.0, False),      # 8-element vector units
    ([(4, 256, 14, 14)] * 2, True, 0.0, False),      # 196 % 8 == 4: masked 8-element covers
    ([(3, 128, 7, 7), (1, 128, 7, 7)], False, 3.0, False),  # odd planes, unequal shards
    ([(2, 32, 3, 3)] * 2, False, 0.0, False),        # scalar units (HW < 16)
    ([(2, 64, 28, 28)] * 2, True, 0.0, True),        # channels_last, C % 8 == 0
    ([(2, 12, 10, 10)] * 2, False, 0.0, True),       # channels_last, C % 8 != 0
])
def test_half_parity(dtype, shapes, relu, loc, cl):
    xs, dys, gamma, beta, ref = _case(shapes, dtype, seed=sum(shapes[0]) + len(shapes), loc=loc,
                                      relu=relu)
    outs = _run(xs, dys, gamma, beta, relu=relu, channels_last=cl)
    tol = OUT_TOL[dtype]
    for r, o in enumerate(outs):
        for key in ("mu", "var", "running_mean", "running_var"):
            assert O.rel_err(o[key], ref[r][key]) <= 1e-5, (key, r)
        for key in ("dgamma", "dbeta"):
            assert O.rel_err(o[key], ref[r][key]) <= 1e-4, (key, r)
        # the oracle's y / dx, rounded to the activation dtype, is the best a correct
        # kernel can produce
        for key in ("y", "x_hat", "dx"):
            want = torch.from_numpy(ref[r][key]).to(dtype).double().numpy()
            assert O.rel_err(o[key], want) <= tol, (key, r, O.rel_err(o[key], want))
    assert np.array_equal(outs[0]["mu"], outs[-1]["mu"])


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_half_two_d_and_eval(dtype):
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal((64, 40)).astype(np.float32)).to(dtype).to(dev)
    st = cg.BNLayerState(gamma=np.ones(40), beta=np.zeros(40))
    y, cache = cg.bn_forward_local(x, st)
    xd = x.double().cpu().numpy()
    mu, var = xd.mean(0), xd.var(0)
    assert O.rel_err(cache.mu.cpu().numpy(), mu) <= 1e-5
    want = torch.from_numpy((xd - mu) / np.sqrt(var + 1e-5)).to(dtype).double().numpy()
    assert O.rel_err(y.double().cpu().numpy(), want) <= OUT_TOL[dtype]
    ye, _ = cg.bn_forward_local(x, st, mode="eval")
    assert ye.dtype == dtype


def test_mixed_dtypes_rejected():
    dev = torch.device("cuda", 0)
    x = torch.randn(2, 4, 5, 5, device=dev, dtype=torch.bfloat16)
    st = cg.BNLayerState(gamma=np.ones(4), beta=np.zeros(4))
    _, cache = cg.bn_forward_local(x, st)
    with pytest.raises(cg.BatchNormError, match="dtype"):
        cg.bn_backward_local(torch.randn(2, 4, 5, 5, device=dev), cache, st)
    with pytest.raises(cg.TensorError):
        cg.channel_sum(torch.randn(2, 4, device=dev, dtype=torch.float64))
