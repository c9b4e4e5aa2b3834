"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors
and the pinned oracle, on the same seeded inputs split identically across ranks.

Tolerances (stated, fp32 path vs the f64 reference; metric = the reference's rel_err,
max|a-b| / max(|a|,|b|,1e-3), pkg/tests/helpers.py:158-163):
    mean, var, y, x_hat, running_mean, running_var : 1e-5
    dx, dgamma, dbeta                              : 1e-4
"""

import numpy as np
import pytest
import torch

from golden_cases import case_names, load_case
from oracle import cgbn_oracle as O

import paper_1711_07240_b200 as cg

pytestmark = pytest.mark.gpu

TOL_FWD = 1e-5
TOL_BWD = 1e-4


def _dev():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    return torch.device("cuda", 0)


def run_group(world, g, xs, dys, gamma, beta, eps=1e-5, momentum=0.1, rm0=None, rv0=None,
              one_pass=False, relu=False, channels_last=False):
    dev = _dev()
    xs_t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in xs]
    dys_t = [torch.from_numpy(np.ascontiguousarray(d)).to(dev) for d in dys] if dys else None
    if channels_last:
        xs_t = [x.contiguous(memory_format=torch.channels_last) for x in xs_t]
        if dys_t:
            dys_t = [d.contiguous(memory_format=torch.channels_last) for d in dys_t]

    def worker(h):
        st = cg.BNLayerState(gamma=gamma, beta=beta, eps=eps, running_mean=rm0,
                             running_var=rv0, running_momentum=momentum)
        y, cache = cg.sync_bn_forward(h, xs_t[h.rank], st, one_pass=one_pass, relu=relu)
        out = dict(y=y, mu=cache.mu, var=cache.var, m=cache.total_count,
                   running_mean=st.running_mean, running_var=st.running_var,
                   x_hat=cache.x_hat)
        if dys_t is not None:
            dx, dgamma, dbeta = cg.sync_bn_backward(h, dys_t[h.rank], cache, st)
            out.update(dx=dx, dgamma=dgamma, dbeta=dbeta)
        return {k: (v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v)
                for k, v in out.items()}

    return cg.DeviceGroup(world, bn_group_size=g, timeout_s=60.0).run(worker)


@pytest.mark.parametrize("name", case_names())
def test_golden_parity(name):
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
        assert o["m"] == int(a[f"m_{r}"])


@pytest.mark.parametrize("name", ["config1_mini", "hw49", "relu", "two_d"])
def test_golden_parity_channels_last(name):
    meta, a = load_case(name)
    if len(meta["shapes"][0]) != 4:
        pytest.skip("2-D input has no channels_last form")
    world = meta["world"]
    outs = run_group(world, meta["bn_group"], [a[f"x_{r}"] for r in range(world)],
                     [a[f"dy_{r}"] for r in range(world)], a["gamma"], a["beta"], meta["eps"],
                     meta["momentum"], a["running_mean0"], a["running_var0"],
                     meta["one_pass"], meta["relu"], channels_last=True)
    for r in range(world):
        for key in ("y", "mu", "var"):
            assert O.rel_err(outs[r][key], a[f"{key}_{r}"]) <= TOL_FWD
        for key in ("dx", "dgamma", "dbeta"):
            assert O.rel_err(outs[r][key], a[f"{key}_{r}"]) <= TOL_BWD


@pytest.mark.parametrize("name", case_names())
def test_golden_eval(name):
    meta, a = load_case(name)
    dev = _dev()
    st = cg.BNLayerState(gamma=a["gamma"], beta=a["beta"], eps=meta["eps"],
                         running_mean=a["running_mean_0"].astype(np.float32),
                         running_var=a["running_var_0"].astype(np.float32),
                         running_momentum=meta["momentum"])
    rm_before = st.running_mean.clone()
    y, cache = cg.bn_forward_local(torch.from_numpy(a["x_0"]).to(dev), st, mode="eval")
    assert O.rel_err(y.cpu().numpy(), a["eval_y_0"]) <= TOL_FWD
    assert torch.equal(st.running_mean, rm_before)  # eval leaves the state untouched
    assert cache.train is False
    with pytest.raises(cg.BatchNormError, match="training-mode"):
        cg.bn_backward_local(torch.from_numpy(a["x_0"]).to(dev), cache, st)


def _oracle_case(shapes, seed, loc=0.0, g=None, relu=False):
    rng = np.random.default_rng(seed)
    c = shapes[0][1]
    xs = [(loc + rng.standard_normal(s)).astype(np.float32) for s in shapes]
    dys = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.standard_normal(c).astype(np.float32)
    g = len(shapes) if g is None else g
    ref = O.cgbn_world([x.astype(np.float64) for x in xs], gamma.astype(np.float64),
                       beta.astype(np.float64), g, relu=relu,
                       dys=[d.astype(np.float64) for d in dys])
    return xs, dys, gamma, beta, g, ref


@pytest.mark.parametrize("shape,world,loc", [
    ((2, 64, 56, 56), 4, 0.0),     # config 1: 4 simulated devices on one GPU
    ((1, 2048, 7, 7), 8, 0.0),     # config 5 shape, G=8 emulated
    ((2, 256, 13, 21), 2, 0.0),    # FPN P6, HW % 4 == 1
    ((2, 256, 25, 42), 2, 3.0),    # FPN P5, HW % 4 == 2, shifted mean
    ((4, 128, 28, 28), 2, 0.0),
    ((2, 64, 56, 56), 2, 1000.0),  # adversarial mean (|mu| >> sigma)
])
def test_oracle_parity_shapes(shape, world, loc):
    xs, dys, gamma, beta, g, ref = _oracle_case([shape] * world, seed=sum(shape) + world,
                                                loc=loc)
    outs = run_group(world, g, xs, dys, gamma, beta)
    for r in range(world):
        for key in ("y", "mu", "var", "running_mean", "running_var"):
            assert O.rel_err(outs[r][key], ref[r][key]) <= TOL_FWD, (key, r)
        for key in ("dx", "dgamma", "dbeta"):
            assert O.rel_err(outs[r][key], ref[r][key]) <= TOL_BWD, (key, r)


@pytest.mark.parametrize("shapes,relu,loc", [
    ([(2, 64, 56, 56)] * 4, False, 0.0),            # config 1 in channels_last
    ([(3, 256, 14, 14), (1, 256, 14, 14)], True, 0.0),  # unequal shards + ReLU
    ([(2, 2048, 7, 7)] * 2, False, 3.0),            # two channel slices, shifted mean
    ([(2, 100, 9, 9)] * 2, True, 0.0),              # C % 4 == 0, odd plane
    ([(2, 30, 5, 5)] * 2, False, 0.0),              # C % 4 != 0: generic path
    ([(4, 64, 56, 56)], False, 1000.0),             # single rank, adversarial mean
])
def test_channels_last_row_kernels(shapes, relu, loc):
    """NHWC activations: the row reductions (k_reduce_rows + k_fold_rows) and the
    channels_last elementwise mode against the oracle."""
    world = len(shapes)
    xs, dys, gamma, beta, g, ref = _oracle_case(shapes, seed=sum(shapes[0]) + world, loc=loc,
                                                relu=relu)
    outs = run_group(world, g, xs, dys, gamma, beta, relu=relu, channels_last=True)
    for r in range(world):
        for key in ("y", "mu", "var", "running_mean", "running_var"):
            assert O.rel_err(outs[r][key], ref[r][key]) <= TOL_FWD, (key, r)
        for key in ("dx", "dgamma", "dbeta"):
            assert O.rel_err(outs[r][key], ref[r][key]) <= TOL_BWD, (key, r)
    for r in range(1, world):
        assert np.array_equal(outs[r]["mu"], outs[0]["mu"])
        assert np.array_equal(outs[r]["dgamma"], outs[0]["dgamma"])


@pytest.mark.parametrize("n,c", [(64, 256), (7, 1024), (33, 12), (5, 3)])
def test_two_d_rows(n, c):
    """(N, C) activations (the reference's 2-D layout) through the row kernels."""
    xs, dys, gamma, beta, g, ref = _oracle_case([(n, c)] * 2, seed=n + c)
    outs = run_group(2, g, xs, dys, gamma, beta)
    for r in range(2):
        for key in ("y", "mu", "var"):
            assert O.rel_err(outs[r][key], ref[r][key]) <= TOL_FWD, (key, r)
        for key in ("dx", "dgamma", "dbeta"):
            assert O.rel_err(outs[r][key], ref[r][key]) <= TOL_BWD, (key, r)


def test_relu_fused_parity_config1():
    xs, dys, gamma, beta, g, ref = _oracle_case([(2, 64, 56, 56)] * 4, seed=7, relu=True)
    outs = run_group(4, g, xs, dys, gamma, beta, relu=True)
    for r in range(4):
        assert O.rel_err(outs[r]["y"], ref[r]["y"]) <= TOL_FWD
        assert O.rel_err(outs[r]["dx"], ref[r]["dx"]) <= TOL_BWD
        assert O.rel_err(outs[r]["dgamma"], ref[r]["dgamma"]) <= TOL_BWD


def test_stats_bitwise_identical_across_ranks():
    # test_batchnorm.py:233-239, 277-287, 398-412
    xs, dys, gamma, beta, g, _ = _oracle_case(
        [(3, 32, 9, 9), (1, 32, 9, 9), (2, 32, 9, 9), (4, 32, 9, 9)], seed=42)
    outs = run_group(4, 4, xs, dys, gamma, beta)
    for r in range(1, 4):
        for key in ("mu", "var", "running_mean", "running_var", "dgamma", "dbeta"):
            assert np.array_equal(outs[r][key], outs[0][key]), key


def test_subgroups_isolated():
    xs, dys, gamma, beta, _, _ = _oracle_case([(2, 8, 5, 5)] * 4, seed=61)
    outs = run_group(4, 2, xs, dys, gamma, beta)
    assert np.array_equal(outs[0]["dgamma"], outs[1]["dgamma"])
    assert np.array_equal(outs[2]["dgamma"], outs[3]["dgamma"])
    assert not np.array_equal(outs[0]["dgamma"], outs[2]["dgamma"])
    assert not np.array_equal(outs[0]["mu"], outs[2]["mu"])


def test_group_of_one_bitwise_equals_local():
    # test_batchnorm.py:241-250
    dev = _dev()
    rng = np.random.default_rng(43)
    x = rng.normal(size=(4, 3, 2, 2)).astype(np.float32)
    outs = run_group(2, 1, [x, rng.normal(size=(4, 3, 2, 2)).astype(np.float32)], None,
                     np.ones(3, np.float32), np.zeros(3, np.float32))
    y_local, cache_local = cg.bn_forward_local(torch.from_numpy(x).to(dev),
                                               cg.BNLayerState.create(3))
    assert np.array_equal(outs[0]["y"], y_local.cpu().numpy())
    assert np.array_equal(outs[0]["mu"], cache_local.mu.cpu().numpy())
    assert np.array_equal(outs[0]["var"], cache_local.var.cpu().numpy())


def test_run_to_run_bitwise():
    xs, dys, gamma, beta, g, _ = _oracle_case([(8, 64, 28, 28)] * 2, seed=5)
    a = run_group(2, 2, xs, dys, gamma, beta)
    b = run_group(2, 2, xs, dys, gamma, beta)
    for r in range(2):
        for key in ("y", "mu", "var", "dx", "dgamma", "dbeta"):
            assert np.array_equal(a[r][key], b[r][key]), key


def test_concat_equivalence_large():
    # Full-size property: 4 shards of [8,64,56,56] == local BN over the concatenation
    xs, dys, gamma, beta, _, _ = _oracle_case([(8, 64, 56, 56)] * 4, seed=9)
    outs = run_group(4, 4, xs, dys, gamma, beta)
    one = run_group(1, 1, [np.concatenate(xs)], [np.concatenate(dys)], gamma, beta)
    y = np.concatenate([o["y"] for o in outs])
    dx = np.concatenate([o["dx"] for o in outs])
    assert O.rel_err(y, one[0]["y"]) <= TOL_FWD
    assert O.rel_err(dx, one[0]["dx"]) <= TOL_BWD
    assert O.rel_err(outs[0]["mu"], one[0]["mu"]) <= 1e-7
    assert O.rel_err(outs[0]["var"], one[0]["var"]) <= 1e-7


def test_errors_match_reference():
    dev = _dev()
    st = cg.BNLayerState.create(3)
    with pytest.raises(cg.BatchNormError, match="at least 2"):
        cg.bn_forward_local(torch.ones((1, 3), device=dev), st)
    with pytest.raises(cg.BatchNormError):
        cg.bn_forward_local(torch.ones((4, 2), device=dev), st)  # channel mismatch
    with pytest.raises(cg.BatchNormError):
        cg.bn_forward_local(torch.ones((4, 3), device=dev), st, mode="test")
    x = torch.randn(4, 3, device=dev)
    x[1, 2] = float("nan")
    with pytest.raises(cg.NonFiniteError):
        cg.bn_forward_local(x, cg.BNLayerState.create(3))
    with pytest.raises(cg.BatchNormError, match="cotangent"):
        _, cache = cg.bn_forward_local(torch.randn(4, 3, device=dev), cg.BNLayerState.create(3))
        cg.bn_backward_local(torch.ones((3, 3), device=dev), cache, cg.BNLayerState.create(3))

    def mismatch(h):
        c = 3 if h.rank == 0 else 4
        return cg.sync_bn_forward(h, torch.ones((2, c), device=dev), cg.BNLayerState.create(c))

    with pytest.raises(cg.CollectiveProtocolError):
        cg.DeviceGroup(2, timeout_s=5.0).run(mismatch)

    def small(h):
        return cg.sync_bn_forward(h, torch.ones((1, 3), device=dev), cg.BNLayerState.create(3))

    with pytest.raises(cg.BatchNormError, match="at least 2"):
        cg.DeviceGroup(1).run(small)

    def foreign(h):
        _, cache = cg.bn_forward_local(torch.randn(4, 2, device=dev), cg.BNLayerState.create(2))
        return cg.sync_bn_backward(h, torch.randn(4, 2, device=dev), cache,
                                   cg.BNLayerState.create(2))

    with pytest.raises(cg.BatchNormError):
        cg.DeviceGroup(1).run(foreign)


def test_inplace_change_of_x_before_backward_raises():
    """The cache holds x by reference (x_hat is recomputed), so an in-place change of x
    between forward and backward must raise instead of giving wrong gradients."""
    dev = _dev()
    x = torch.randn(4, 3, 5, 5, device=dev)
    st = cg.BNLayerState.create(3)
    _, cache = cg.bn_forward_local(x, st)
    x.mul_(2.0)
    with pytest.raises(cg.BatchNormError, match="in place"):
        cg.bn_backward_local(torch.randn_like(x), cache, st)
    _, cache = cg.bn_forward_local(x, st)  # untouched x: fine
    cg.bn_backward_local(torch.randn_like(x), cache, st)


def test_allreduce_sum_ascending_fold_bitwise():
    # collectives.py:293-295 / test_collectives.py:43-51
    dev = _dev()
    vals = [torch.tensor([1e16, -0.0], dtype=torch.float64, device=dev),
            torch.tensor([1.0, -0.0], dtype=torch.float64, device=dev),
            torch.tensor([-1e16, -0.0], dtype=torch.float64, device=dev)]

    def fn(h):
        return cg.allreduce_sum(h, cg.SCOPE_WORLD, vals[h.rank]).cpu().numpy()

    outs = cg.DeviceGroup(3).run(fn)
    for o in outs:
        assert o[0] == 0.0 and np.signbit(o[1])


def test_channel_primitives():
    dev = _dev()
    rng = np.random.default_rng(17)
    x = rng.normal(size=(3, 2, 2, 2)).astype(np.float32)
    st = cg.channel_sum(torch.from_numpy(x).to(dev), with_sum_sq=True)
    cnt, s, ss = O.channel_sum(x.astype(np.float64), with_sum_sq=True)
    assert st.count == cnt
    assert O.rel_err(st.sum.cpu().numpy(), s) <= 1e-12
    assert O.rel_err(st.sum_sq.cpu().numpy(), ss) <= 1e-12
    out = cg.channel_affine(torch.from_numpy(x).to(dev), [2.0, -1.0], [0.5, 0.25])
    want = O.channel_affine(x.astype(np.float64), [2.0, -1.0], [0.5, 0.25])
    assert O.rel_err(out.cpu().numpy(), want) <= 1e-7


def _local_run(x, dy, gamma, beta, relu=False):
    dev = _dev()
    st = cg.BNLayerState(gamma=gamma, beta=beta)
    y, cache = cg.bn_forward_local(torch.from_numpy(x).to(dev), st, relu=relu)
    dx, dgamma, dbeta = cg.bn_backward_local(torch.from_numpy(dy).to(dev), cache, st)
    return dict(y=y.cpu().numpy(), mu=cache.mu.cpu().numpy(), var=cache.var.cpu().numpy(),
                running_mean=st.running_mean.cpu().numpy(),
                running_var=st.running_var.cpu().numpy(), dx=dx.cpu().numpy(),
                dgamma=dgamma.cpu().numpy(), dbeta=dbeta.cpu().numpy())


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("shape,loc,relu", [
    ((8, 64, 28, 28), 0.0, False),
    ((4, 256, 14, 14), 2.0, True),
    ((32, 128, 28, 28), 0.0, False),   # 3.2M elements: fused forward and backward
    ((32, 64, 56, 56), -5.0, False),   # 6.4M: fused forward only (backward split)
    ((3, 5, 4, 8), 0.0, True),         # tiny, one CTA
])
def test_single_rank_fused_and_split(shape, loc, relu, fused):
    prev = cg.set_fused(fused)
    try:
        xs, dys, gamma, beta, _, ref = _oracle_case([shape], seed=sum(shape), loc=loc, relu=relu)
        out = _local_run(xs[0], dys[0], gamma, beta, relu=relu)
    finally:
        cg.set_fused(prev)
    for key in ("y", "mu", "var", "running_mean", "running_var"):
        assert O.rel_err(out[key], ref[0][key]) <= TOL_FWD, key
    for key in ("dx", "dgamma", "dbeta"):
        assert O.rel_err(out[key], ref[0][key]) <= TOL_BWD, key


def test_fused_eligibility():
    from paper_1711_07240_b200 import _lib
    _dev()
    lib = _lib.load()
    assert lib.cgbn_fused_supported(32, 128, 784, 0, 0) == 1
    assert lib.cgbn_fused_supported(32, 128, 784, 0, 1) == 1
    assert lib.cgbn_fused_supported(32, 64, 3136, 0, 0) == 1
    assert lib.cgbn_fused_supported(32, 64, 3136, 0, 1) == 0      # 6.4M: backward too big
    assert lib.cgbn_fused_supported(32, 256, 3136, 0, 0) == 0     # 25.7M: neither
    assert lib.cgbn_fused_supported(32, 2048, 49, 0, 0) == 1      # odd planes: lead-aware path
    assert lib.cgbn_fused_supported(32, 2048, 49, 0, 1) == 1
    assert lib.cgbn_fused_supported(32, 128, 784, 1, 0) == 0      # NHWC
    # the automatic choice of the *_local / statistics entry points (in-step footprint cap)
    assert lib.cgbn_onchip_selected(32, 128, 784, 0, 0) == 1      # 12.8 MB forward
    assert lib.cgbn_onchip_selected(32, 128, 784, 0, 1) == 0      # 25.7 MB backward
    assert lib.cgbn_onchip_selected(32, 64, 3136, 0, 0) == 0
    assert lib.cgbn_onchip_selected(32, 256, 196, 0, 1) == 1
    assert lib.cgbn_onchip_selected(32, 256, 196, _lib.ACT_BF16, 0) == 0  # 16-bit: off
    assert lib.cgbn_onchip_selected(1, 2048, 49, 0, 0) == 0       # one image: split path
    assert lib.cgbn_fused_supported(1, 2048, 49, 0, 0) == 1       # (forced: still on chip)


def test_fused_run_to_run_bitwise_and_matches_split_closely():
    xs, dys, gamma, beta, _, _ = _oracle_case([(16, 96, 28, 28)], seed=77)
    a = _local_run(xs[0], dys[0], gamma, beta)
    b = _local_run(xs[0], dys[0], gamma, beta)
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    prev = cg.set_fused(False)
    try:
        s = _local_run(xs[0], dys[0], gamma, beta)
    finally:
        cg.set_fused(prev)
    assert O.rel_err(a["mu"], s["mu"]) <= 1e-9
    assert O.rel_err(a["y"], s["y"]) <= 1e-6


@pytest.mark.parametrize("layout,dtype", [("nchw", torch.float32), ("nhwc", torch.float32),
                                          ("nchw", torch.bfloat16), ("2d", torch.float32)])
def test_nonfinite_detected_every_path(layout, dtype):
    """NaN in x is reported as NonFiniteError through every reduction path (cluster-team,
    rows, 16-bit), and Inf in dy through the backward (tensor.py:59-60)."""
    dev = _dev()
    shape = (4, 32) if layout == "2d" else (2, 8, 6, 6)
    x = torch.randn(shape, device=dev).to(dtype)
    if layout == "nhwc":
        x = x.contiguous(memory_format=torch.channels_last)
    x[(1, 2) if layout == "2d" else (1, 2, 3, 4)] = float("nan")
    c = shape[1]
    st = cg.BNLayerState(gamma=np.ones(c), beta=np.zeros(c))
    with pytest.raises(cg.NonFiniteError):
        cg.bn_forward_local(x, st)
    x2 = torch.randn(shape, device=dev).to(dtype)
    if layout == "nhwc":
        x2 = x2.contiguous(memory_format=torch.channels_last)
    st = cg.BNLayerState(gamma=np.ones(c), beta=np.zeros(c))
    _, cache = cg.bn_forward_local(x2, st)
    dy = torch.randn(shape, device=dev).to(dtype)
    if layout == "nhwc":
        dy = dy.contiguous(memory_format=torch.channels_last)
    dy[(0, 3) if layout == "2d" else (0, 5, 1, 2)] = float("inf")
    with pytest.raises(cg.NonFiniteError):
        cg.bn_backward_local(dy, cache, st)


def test_world_mean_allreduce_matches_trainer_step():
    """trainer.py:419-428: sorted-key concatenation + loss, ascending fold / world, split
    back; bitwise identical on every rank (float32 fold in rank order)."""
    dev = _dev()
    rng = np.random.default_rng(11)
    world = 4
    shapes = {"b.w": (3, 5), "a.gamma": (7,), "c.b": (2, 2, 2)}
    grads = [{k: rng.standard_normal(s).astype(np.float32) for k, s in shapes.items()}
             for _ in range(world)]
    losses = [float(rng.standard_normal()) for _ in range(world)]

    def worker(h):
        g = {k: torch.from_numpy(v).to(dev) for k, v in grads[h.rank].items()}
        mean, loss = cg.world_mean_allreduce(h, g, losses[h.rank])
        return {k: v.cpu().numpy() for k, v in mean.items()}, loss

    out = cg.DeviceGroup(world, timeout_s=60.0).run(worker)
    keys = sorted(shapes)
    flat = [np.concatenate([grads[r][k].ravel() for k in keys] + [np.array([losses[r]], np.float32)])
            for r in range(world)]
    acc = flat[0].copy()
    for f in flat[1:]:
        acc = acc + f
    want = acc / np.float32(world)
    off = 0
    for k in keys:
        n = int(np.prod(shapes[k]))
        for r in range(world):
            assert np.array_equal(out[r][0][k].ravel(), want[off:off + n]), (k, r)
        off += n
    assert all(out[r][1] == float(want[-1]) for r in range(world))


@pytest.mark.parametrize("shape,cl", [
    ((1, 65535, 2, 2), False),   # C at the ABI limit: cluster-team clusters loop over groups
    ((2, 8192, 3, 3), False),    # masked-free scalar units, looping clusters
    ((2, 65532, 1, 1), True),    # channels_last rows kernel: 64 channel slices
    ((3, 65535), False),         # 2-D with C % 4 != 0 (team fallback)
])
def test_max_channels(shape, cl):
    """The widest layers (C up to 65535, include/cgbn.h) through every decomposition."""
    xs, dys, gamma, beta, g, ref = _oracle_case([shape] * 2, seed=5)
    outs = run_group(2, g, xs, dys, gamma, beta, channels_last=cl and len(shape) == 4)
    for r in range(2):
        for key in ("y", "mu", "var", "running_var"):
            assert O.rel_err(outs[r][key], ref[r][key]) <= TOL_FWD, (key, r)
        for key in ("dx", "dgamma", "dbeta"):
            assert O.rel_err(outs[r][key], ref[r][key]) <= TOL_BWD, (key, r)


@pytest.mark.parametrize("cl", [False, True])
def test_misaligned_view_is_realigned(cl):
    """A contiguous view with an unaligned storage offset runs (copied to aligned
    storage by tensor.geometry) and matches the oracle (VERDICT r1 hygiene)."""
    dev = _dev()
    rng = np.random.default_rng(77)
    if cl:
        base = torch.from_numpy(rng.standard_normal(4 * 4 * 4 * 3 + 1).astype(np.float32))
        x = base.to(dev)[1:].view(4, 4, 4, 3).permute(0, 3, 1, 2)  # NHWC storage
        assert x.is_contiguous(memory_format=torch.channels_last)
    else:
        base = torch.from_numpy(rng.standard_normal((9, 3)).astype(np.float32)).to(dev)
        x = base[1:]
    assert x.data_ptr() % 16 != 0
    st = cg.BNLayerState.create(3)
    y, cache = cg.bn_forward_local(x, st)
    dx, dg, db = cg.bn_backward_local(torch.ones_like(x), cache, st)
    ref = O.cgbn_world([x.double().cpu().numpy()], np.ones(3), np.zeros(3), 1,
                       dys=[np.ones(tuple(x.shape))])[0]
    assert O.rel_err(y.cpu().numpy(), ref["y"]) <= TOL_FWD
    assert O.rel_err(dx.cpu().numpy(), ref["dx"]) <= TOL_BWD
