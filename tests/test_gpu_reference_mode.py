"""set_forward_exchange("reference"): the reference's own statistics arithmetic on the
device (batchnorm.py:118-132), checked against the golden vectors the
real reference produced, plus the exchange count of each mode (two collectives per
two-pass forward, one per one-pass or merged forward) and bitwise rank symmetry.

Tolerances as in test_gpu_parity.py (rel_err with the reference's 1e-3 floor):
    mean, var, y, x_hat, running stats 1e-5; dx, dgamma, dbeta 1e-4.
"""

import numpy as np
import pytest
import torch

from golden_cases import case_names, load_case
from oracle import cgbn_oracle as O
from test_gpu_parity import TOL_BWD, TOL_FWD, run_group

import paper_1711_07240_b200 as cg

pytestmark = pytest.mark.gpu


@pytest.fixture
def reference_mode():
    prev = cg.set_forward_exchange("reference")
    yield
    cg.set_forward_exchange(prev)


@pytest.mark.parametrize("name", case_names())
def test_golden_parity_reference_mode(name, reference_mode):
    meta, a = load_case(name)
    world = meta["world"]
    xs = [a[f"x_{r}"] for r in range(world)]
    dys = [a[f"dy_{r}"] for r in range(world)]
    outs = run_group(world, meta["bn_group"], xs, dys, a["gamma"], a["beta"], meta["eps"],
                     meta["momentum"], a["running_mean0"], a["running_var0"],
                     meta["one_pass"], meta["relu"])
    for r in range(world):
        o = outs[r]
        for key in ("y", "mu", "var", "x_hat", "running_mean", "running_var"):
            e = O.rel_err(o[key], a[f"{key}_{r}"])
            assert e <= TOL_FWD, (name, r, key, e)
        for key in ("dx", "dgamma", "dbeta"):
            e = O.rel_err(o[key], a[f"{key}_{r}"])
            assert e <= TOL_BWD, (name, r, key, e)


class _Counting:
    """Wraps a DeviceHandle and counts forward exchanges."""

    def __init__(self, h):
        self._h = h
        self.n = 0

    def __getattr__(self, k):
        return getattr(self._h, k)

    def exchange(self, scope, kind, vec, info=None):
        if kind == "bn_forward":
            self.n += 1
        return self._h.exchange(scope, kind, vec, info)


@pytest.mark.parametrize("mode,one_pass,want", [
    ("reference", False, 2), ("reference", True, 1), ("merged", False, 1), ("merged", True, 1)])
def test_exchange_count_per_mode(mode, one_pass, want):
    prev = cg.set_forward_exchange(mode)
    try:
        dev = torch.device("cuda", 0)
        rng = np.random.default_rng(5)
        xs = [torch.from_numpy(rng.standard_normal((2, 8, 6, 6)).astype(np.float32)).to(dev)
              for _ in range(2)]

        def worker(h):
            ch = _Counting(h)
            st = cg.BNLayerState(gamma=np.ones(8), beta=np.zeros(8))
            y, cache = cg.sync_bn_forward(ch, xs[h.rank], st, one_pass=one_pass)
            return ch.n, cache.mu.cpu().numpy(), cache.var.cpu().numpy()

        out = cg.DeviceGroup(2, timeout_s=60.0).run(worker)
        assert out[0][0] == want and out[1][0] == want
        # bitwise identical statistics on both ranks
        assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])
        cat = np.concatenate([x.cpu().numpy() for x in xs]).astype(np.float64)
        assert O.rel_err(out[0][1], cat.mean(axis=(0, 2, 3))) <= TOL_FWD
        assert O.rel_err(out[0][2], cat.var(axis=(0, 2, 3))) <= TOL_FWD
    finally:
        cg.set_forward_exchange(prev)


def test_reference_and_merged_modes_agree():
    """Both modes compute the same statistics to fp64 rounding at a shifted mean."""
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(9)
    x = torch.from_numpy((rng.standard_normal((4, 16, 12, 12)) + 3.0).astype(np.float32)).to(dev)
    res = {}
    for mode in ("merged", "reference"):
        prev = cg.set_forward_exchange(mode)
        try:
            st = cg.BNLayerState(gamma=np.ones(16), beta=np.zeros(16))
            y, cache = cg.bn_forward_local(x, st)
            res[mode] = (y.cpu().numpy(), cache.mu.cpu().numpy(), cache.var.cpu().numpy())
        finally:
            cg.set_forward_exchange(prev)
    for a, b in zip(res["merged"], res["reference"]):
        assert O.rel_err(a, b) <= 1e-6


def test_set_forward_exchange_validates():
    with pytest.raises(ValueError):
        cg.set_forward_exchange("nope")
