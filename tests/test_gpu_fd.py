"""Gradient check of the CGBN backward by central differences (the reference's acceptance
criterion C2, `pkg/tests/test_acceptance.py:89-160`, and `verify.py:149-214`), plus the
mutation test that proves the check has teeth (`verify.py:267-278`,
`test_cli.py:169-175`).

The objective is L = sum_r <y_r, w_r> over every rank of the world, with y the cross-GPU
BN forward of the sharded batch. Its central differences are taken on the oracle's f64
forward (`oracle.cgbn_oracle.cgbn_world`, which restates `batchnorm.py:115-144`), so they
share no code with the backward formula of either implementation. The GPU backward
(`sync_bn_backward` with dy = w, through the C ABI) must match them: dx on sampled
entries of every shard, dgamma / dbeta (BN-group sums, `batchnorm.py:203`) on every
channel. Tolerance: normwise 1e-4 (fp32 gradients, `north_star`); the reference's 1e-6
is for its f64 arithmetic.

Mutation: the same backward with eps = 3e-3 instead of the forward's 1e-5 must FAIL the
check, as in the reference's verify suite."""

import numpy as np
import pytest
import torch

from oracle import cgbn_oracle as O

import paper_1711_07240_b200 as cg

pytestmark = pytest.mark.gpu

TOL = 1e-4
H = 1e-4


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    world = [1, 2, 3, 4][seed % 4]
    g = world if seed % 3 else max(1, world // 2 if world % 2 == 0 else world)
    c = int(rng.integers(2, 6))
    spatial = [] if seed % 5 == 4 else [int(rng.integers(1, 5)), int(rng.integers(1, 5))]
    # unequal shards; at least 2 elements per channel in every BN group
    ns = [int(rng.integers(1, 4)) for _ in range(world)]
    if int(np.prod(spatial or [1])) * min(ns) < 2:
        ns = [n + 1 for n in ns]
    xs = [rng.normal(0.5, 1.5, size=(n, c, *spatial)).astype(np.float32) for n in ns]
    ws = [rng.normal(size=x.shape).astype(np.float32) for x in xs]
    gamma = rng.uniform(0.5, 1.5, size=c).astype(np.float32)
    beta = rng.normal(size=c).astype(np.float32)
    return world, g, xs, ws, gamma, beta


def _objective(xs, ws, gamma, beta, g):
    outs = O.cgbn_world([np.asarray(x, np.float64) for x in xs],
                        np.asarray(gamma, np.float64), np.asarray(beta, np.float64), g)
    return sum(float(np.sum(o["y"] * w.astype(np.float64))) for o, w in zip(outs, ws))


def _gpu_backward(world, g, xs, ws, gamma, beta, bwd_eps=1e-5):
    dev = torch.device("cuda", 0)
    xs_t = [torch.from_numpy(x).to(dev) for x in xs]
    ws_t = [torch.from_numpy(w).to(dev) for w in ws]

    def worker(h):
        st = cg.BNLayerState(gamma=gamma, beta=beta, eps=1e-5)
        _, cache = cg.sync_bn_forward(h, xs_t[h.rank], st)
        st.eps = bwd_eps  # mutation hook: the backward reads state.eps (batchnorm.py:205)
        dx, dgamma, dbeta = cg.sync_bn_backward(h, ws_t[h.rank], cache, st)
        return dx.cpu().numpy(), dgamma.cpu().numpy(), dbeta.cpu().numpy()

    return cg.DeviceGroup(world, bn_group_size=g, timeout_s=60.0).run(worker)


def _normwise(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-3))


def _fd_errors(seed, bwd_eps=1e-5):
    world, g, xs, ws, gamma, beta = _case(seed)
    outs = _gpu_backward(world, g, xs, ws, gamma, beta, bwd_eps)
    rng = np.random.default_rng(seed)
    got, fd = [], []
    for r in range(world):
        flat = xs[r].reshape(-1)
        for i in rng.choice(flat.size, size=min(6, flat.size), replace=False):
            xp = [x.copy() for x in xs]
            xm = [x.copy() for x in xs]
            # the oracle runs in f64, so the perturbation is applied to the f64 cast
            xp[r] = xp[r].astype(np.float64)
            xm[r] = xm[r].astype(np.float64)
            xp[r].reshape(-1)[i] += H
            xm[r].reshape(-1)[i] -= H
            fd.append((_objective(xp, ws, gamma, beta, g)
                       - _objective(xm, ws, gamma, beta, g)) / (2 * H))
            got.append(outs[r][0].reshape(-1)[i])
    err_dx = _normwise(got, fd)
    err_gb = 0.0
    if g == world:  # one BN group: dL/dgamma = the group-summed dgamma every rank holds
        c = gamma.size
        fg, fb = np.zeros(c), np.zeros(c)
        for k in range(c):
            e = np.zeros(c)
            e[k] = H
            g64, b64 = gamma.astype(np.float64), beta.astype(np.float64)
            fg[k] = (_objective(xs, ws, g64 + e, b64, g)
                     - _objective(xs, ws, g64 - e, b64, g)) / (2 * H)
            fb[k] = (_objective(xs, ws, g64, b64 + e, g)
                     - _objective(xs, ws, g64, b64 - e, g)) / (2 * H)
        err_gb = max(_normwise(outs[0][1], fg), _normwise(outs[0][2], fb))
    return err_dx, err_gb


@pytest.mark.parametrize("seed", range(16))
def test_backward_matches_central_differences(seed):
    err_dx, err_gb = _fd_errors(seed)
    assert err_dx <= TOL, f"dx vs central differences: {err_dx:.3g}"
    assert err_gb <= TOL, f"dgamma/dbeta vs central differences: {err_gb:.3g}"


@pytest.mark.parametrize("seed", [1, 2, 5])
def test_mutated_backward_fails_the_check(seed):
    """A backward run with eps = 3e-3 (forward 1e-5) must be caught."""
    err_dx, _ = _fd_errors(seed, bwd_eps=3e-3)
    assert err_dx > TOL, f"the mutation passed the gradient check ({err_dx:.3g})"
