"""More of the reference's CGBN invariants (`pkg/tests/test_batchnorm.py`), on the GPU
path through the C ABI, in both forward-exchange modes:

* identical shards give the single-shard statistics (`:252-261`): with every rank holding
  the same shard, the group mean / variance equal the local ones and every rank's y is
  the same, bitwise;
* one-pass is close to two-pass on loc = 2 data (`:263-275`; the reference's 1e-9 is
  for f64, here the fp32 forward tolerance 1e-5);
* running statistics with momentum 1 are identical on every rank and equal the
  concatenated batch's mean and unbiased variance (`:277-287`)."""

import numpy as np
import pytest
import torch

from oracle import cgbn_oracle as O

import paper_1711_07240_b200 as cg

pytestmark = pytest.mark.gpu

TOL_FWD = 1e-5


@pytest.fixture(params=["merged", "reference"])
def exchange_mode(request):
    prev = cg.set_forward_exchange(request.param)
    yield request.param
    cg.set_forward_exchange(prev)


def _forward(world, g, xs, momentum=0.1, one_pass=False):
    dev = torch.device("cuda", 0)
    xs_t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in xs]
    c = xs[0].shape[1]

    def worker(h):
        st = cg.BNLayerState.create(c, running_momentum=momentum)
        y, cache = cg.sync_bn_forward(h, xs_t[h.rank], st, one_pass=one_pass)
        return {k: v.cpu().numpy() for k, v in dict(
            y=y, mu=cache.mu, var=cache.var, rm=st.running_mean, rv=st.running_var).items()}

    return cg.DeviceGroup(world, bn_group_size=g, timeout_s=60.0).run(worker)


def _local(x):
    dev = torch.device("cuda", 0)
    y, cache = cg.bn_forward_local(torch.from_numpy(np.ascontiguousarray(x)).to(dev),
                                   cg.BNLayerState.create(x.shape[1]))
    return y.cpu().numpy(), cache.mu.cpu().numpy(), cache.var.cpu().numpy()


@pytest.mark.parametrize("shape", [(5, 2), (3, 16, 7, 7), (2, 64, 28, 28)])
def test_identical_shards_give_local_stats(shape, exchange_mode):
    x = np.random.default_rng(44).normal(size=shape).astype(np.float32)
    out = _forward(2, 2, [x, x.copy()])
    _, mu, var = _local(x)
    assert np.array_equal(out[0]["mu"], mu)
    assert np.array_equal(out[0]["var"], var)
    assert np.array_equal(out[0]["y"], out[1]["y"])


@pytest.mark.parametrize("shape", [(3, 4, 2, 2), (2, 32, 14, 14)])
def test_one_pass_close_to_two_pass(shape, exchange_mode):
    rng = np.random.default_rng(45)
    shards = [(2.0 + rng.standard_normal(shape)).astype(np.float32) for _ in range(3)]
    two = _forward(3, 3, shards, one_pass=False)
    one = _forward(3, 3, shards, one_pass=True)
    for r in range(3):
        assert O.rel_err(one[r]["y"], two[r]["y"]) < TOL_FWD


@pytest.mark.parametrize("shape", [(3, 2), (2, 8, 5, 5)])
def test_running_stats_identical_and_unbiased(shape, exchange_mode):
    rng = np.random.default_rng(46)
    shards = [rng.standard_normal(shape).astype(np.float32) for _ in range(2)]
    out = _forward(2, 2, shards, momentum=1.0)
    assert np.array_equal(out[0]["rm"], out[1]["rm"])
    assert np.array_equal(out[0]["rv"], out[1]["rv"])
    concat = np.concatenate(shards).astype(np.float64)
    axes = (0,) + tuple(range(2, concat.ndim))
    m = concat.size // concat.shape[1]
    ref_mu = concat.mean(axis=axes)
    ref_var_unbiased = concat.var(axis=axes) * m / (m - 1)
    assert O.rel_err(out[0]["rm"], ref_mu) <= TOL_FWD
    assert O.rel_err(out[0]["rv"], ref_var_unbiased) <= TOL_FWD
