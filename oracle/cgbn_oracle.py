"""CGBN oracle — TEST INFRASTRUCTURE ONLY.

A CPU (numpy, float64) restatement of the reference algorithm for the CGBN hot path
(/root/reference/pkg/src/bigbatch). Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it, and only as
the checker or the timed CPU baseline — never as part of the product path, which has no
CPU fallback.

Parity pinning: this restatement is checked against (1) the frozen literals of the
reference's own unit tests (test_batchnorm.py:86-97, test_tensor.py:133-156) and
(2) golden vectors produced by running the real reference (tests/golden/make_golden.py
imports /root/reference/pkg/src/bigbatch and writes tests/golden/*.npz); see
tests/test_oracle.py. The arithmetic lives in NumPy (numpy>=1.24 per
pkg/pyproject.toml:9-10; 2.3.5 here): np.cumsum left fold, broadcasting * and +, np.sqrt.

Every function cites the reference lines it restates.
"""

from __future__ import annotations

import numpy as np


# -- tensor.py ---------------------------------------------------------------------

def channels_last_rows(a: np.ndarray) -> np.ndarray:
    """(N,C) or (N,C,H,W) -> (rows, C), sample-major then h then w (tensor.py:121-128)."""
    if a.ndim == 2:
        return a
    if a.ndim == 4:
        n, c, h, w = a.shape
        return a.transpose(0, 2, 3, 1).reshape(n * h * w, c)
    raise ValueError(f"expected layout (N,C) or (N,C,H,W), got rank {a.ndim}")


def sequential_sum_rows(rows: np.ndarray) -> np.ndarray:
    """Strict left fold row 0, row 1, ... in the input dtype (tensor.py:131-140)."""
    if rows.shape[0] == 1:
        return rows[0].copy()
    return np.cumsum(rows, axis=0)[-1]


def channel_sum(x: np.ndarray, with_sum_sq: bool = False):
    """(count, sum, sum_sq|None) per channel (tensor.py:143-153)."""
    rows = channels_last_rows(x)
    s = sequential_sum_rows(rows)
    ss = sequential_sum_rows(rows * rows) if with_sum_sq else None
    return rows.shape[0], s, ss


def channel_affine(x: np.ndarray, scale, shift) -> np.ndarray:
    """out[n,c,...] = scale[c]*x + shift[c], coefficients cast to x's dtype
    (tensor.py:156-170)."""
    c = x.shape[1]
    scale = np.asarray(scale, dtype=x.dtype)
    shift = np.asarray(shift, dtype=x.dtype)
    bshape = (1, c) + (1,) * (x.ndim - 2)
    return scale.reshape(bshape) * x + shift.reshape(bshape)


# -- collectives.py ----------------------------------------------------------------

def star_allreduce(vectors):
    """Root fold in ascending rank order: acc = v[0]; acc = acc + v[r]
    (collectives.py:293-295). Returns the vector every rank receives."""
    acc = np.asarray(vectors[0]).copy()
    for v in vectors[1:]:
        acc = acc + np.asarray(v)
    return acc


# -- batchnorm.py ------------------------------------------------------------------

def update_running(running_mean, running_var, momentum, mu, var, count):
    """bn_update_running (batchnorm.py:239-252): unbiased count/(count-1) on var."""
    if count <= 1:
        raise ValueError(f"running-variance update needs count > 1, got {count}")
    unbiased = var * (count / (count - 1.0))
    return ((1.0 - momentum) * running_mean + momentum * mu,
            (1.0 - momentum) * running_var + momentum * unbiased)


class RankState:
    """One rank's mutable BN state (batchnorm.py:36-87 BNLayerState fields)."""

    def __init__(self, gamma, beta, eps=1e-5, running_mean=None, running_var=None,
                 momentum=0.1):
        c = len(gamma)
        self.gamma = np.asarray(gamma, dtype=np.float64)
        self.beta = np.asarray(beta, dtype=np.float64)
        self.eps = float(eps)
        self.running_mean = (np.zeros(c) if running_mean is None
                             else np.asarray(running_mean, dtype=np.float64).copy())
        self.running_var = (np.ones(c) if running_var is None
                            else np.asarray(running_var, dtype=np.float64).copy())
        self.momentum = float(momentum)


def group_train_forward(shards, states, one_pass: bool = False, relu: bool = False):
    """_train_forward (batchnorm.py:115-144) run in lockstep on the ranks of ONE BN
    group, with reduce_vec = star_allreduce over the group (batchnorm.py:181-185).

    ``shards[r]`` is rank r's (N_r, C[, H, W]) float64 array, ``states[r]`` its
    RankState (updated in place). Returns per-rank dicts with y, x_hat, mu, var, m.
    ``relu`` applies the ReLU that follows BN in the reference model (model.py:243-246).
    """
    c = states[0].gamma.shape[0]
    locs = [channel_sum(x, with_sum_sq=one_pass) for x in shards]
    if one_pass:
        total = star_allreduce([np.concatenate([s, ss, [float(cnt)]])
                                for cnt, s, ss in locs])
        s, ssq, m = total[:c], total[c:2 * c], total[2 * c]
        mu = s / m
        var = np.maximum(ssq / m - mu * mu, 0.0)
    else:
        total = star_allreduce([np.concatenate([s, [float(cnt)]]) for cnt, s, _ in locs])
        s, m = total[:c], total[c]
        mu = s / m
        devs = []
        for x in shards:
            diff = x - mu.reshape((1, c) + (1,) * (x.ndim - 2))
            devs.append(sequential_sum_rows(channels_last_rows(diff * diff)))
        var = star_allreduce(devs) / m
    m_int = int(round(m))
    if m_int < 2:
        raise ValueError(
            f"training-mode statistics need at least 2 elements per channel, got {m_int}")
    inv_std = 1.0 / np.sqrt(var + states[0].eps)
    out = []
    for x, st in zip(shards, states):
        x_hat = channel_affine(x, inv_std, -mu * inv_std)
        y = channel_affine(x_hat, st.gamma, st.beta)
        mask = None
        if relu:
            mask = y > 0
            y = y * mask
        st.running_mean, st.running_var = update_running(
            st.running_mean, st.running_var, st.momentum, mu, var, m_int)
        out.append(dict(y=y, x_hat=x_hat, mu=mu, var=var, m=m_int, mask=mask))
    return out


def group_backward(dys, caches, states):
    """_backward_core (batchnorm.py:188-210) in lockstep over one BN group with
    reduce_vec = star_allreduce. ``caches`` are the per-rank dicts returned by
    group_train_forward. Returns per-rank (dx, dgamma, dbeta); dgamma/dbeta are the
    group sums (batchnorm.py:203)."""
    c = states[0].gamma.shape[0]
    packed = []
    gs = []
    for dy, cache in zip(dys, caches):
        g = dy * cache["mask"] if cache["mask"] is not None else dy
        gs.append(g)
        packed.append(np.concatenate([
            sequential_sum_rows(channels_last_rows(g)),
            sequential_sum_rows(channels_last_rows(g * cache["x_hat"]))]))
    total = star_allreduce(packed)
    dbeta, dgamma = total[:c], total[c:]
    out = []
    for g, cache, st in zip(gs, caches, states):
        m = float(cache["m"])
        inv_std = st.gamma / np.sqrt(cache["var"] + st.eps)
        bshape = (1, c) + (1,) * (g.ndim - 2)
        dx = inv_std.reshape(bshape) * (
            g - dbeta.reshape(bshape) / m - cache["x_hat"] * dgamma.reshape(bshape) / m)
        out.append((dx, dgamma.copy(), dbeta.copy()))
    return out


def eval_forward(x, st: RankState, relu: bool = False):
    """bn_forward_local(mode="eval") (batchnorm.py:158-166)."""
    inv_std = 1.0 / np.sqrt(st.running_var + st.eps)
    x_hat = channel_affine(x, inv_std, -st.running_mean * inv_std)
    y = channel_affine(x_hat, st.gamma, st.beta)
    return y * (y > 0) if relu else y


def cgbn_world(shards, gammas, betas, bn_group_size, one_pass=False, relu=False, dys=None,
               eps=1e-5, momentum=0.1, running=None):
    """Whole-world driver: contiguous BN sub-groups of ``bn_group_size`` ranks
    (collectives.py:98-126), each running group_train_forward (+ group_backward when
    ``dys`` is given). Returns per-rank result dicts (y, mu, var, m, running_mean,
    running_var[, dx, dgamma, dbeta])."""
    world = len(shards)
    if world % bn_group_size:
        raise ValueError("bn_group_size must divide the world size")
    results = [None] * world
    for gi in range(world // bn_group_size):
        ranks = list(range(gi * bn_group_size, (gi + 1) * bn_group_size))
        states = []
        for r in ranks:
            rm, rv = (None, None) if running is None else running
            states.append(RankState(gammas, betas, eps, rm, rv, momentum))
        fwd = group_train_forward([shards[r] for r in ranks], states, one_pass, relu)
        bwd = None
        if dys is not None:
            bwd = group_backward([dys[r] for r in ranks], fwd, states)
        for k, r in enumerate(ranks):
            res = dict(fwd[k])
            res["running_mean"] = states[k].running_mean
            res["running_var"] = states[k].running_var
            if bwd is not None:
                res["dx"], res["dgamma"], res["dbeta"] = bwd[k]
            results[r] = res
    return results


def group_blocks(shards, gamma, beta, dys=None, eps=1e-5, momentum=0.1, relu=False,
                 running=None, block_elems=1 << 25):
    """The same BN group arithmetic as ``group_train_forward`` (two-pass, the reference
    default) + ``group_backward``, for activations too large for the literal
    restatement: channel blocks of at most ``block_elems`` elements per rank, f64.

    Per-channel sums use NumPy's pairwise ``np.add.reduce`` instead of the reference's
    ``np.cumsum`` left fold (tensor.py:131-140). In f64 both are within n * 2^-53 of the
    exact sum (n <= 4.3M terms here: < 5e-10 relative), five orders of magnitude below
    the 1e-5 / 1e-4 fp32 parity tolerances; the group fold over ranks stays ascending
    (collectives.py:293-295). The arithmetic per element is batchnorm.py:125-141
    (mean, centred variance, x_hat = x*inv_std + (-mu*inv_std), y = gamma*x_hat + beta,
    ReLU mask), batchnorm.py:239-252 (running update, m/(m-1)) and batchnorm.py:198-209
    (dbeta = sum g, dgamma = sum g*x_hat, dx).

    ``shards`` / ``dys``: per-rank (N_r, C, H, W) or (N_r, C) arrays (any float dtype;
    promoted to f64 per block). Yields, per channel block, a dict with "c0", "c1",
    group "mu", "var", "m", "running_mean", "running_var" (block slices), and per-rank
    lists "y", "dx" (f64 block arrays, shape (N_r, c1-c0, ...)) plus group "dgamma",
    "dbeta" when ``dys`` is given.
    """
    c = shards[0].shape[1]
    per_c = max(int(np.prod(x.shape)) // c for x in shards)
    step = max(1, min(c, block_elems // max(per_c, 1)))
    m = float(sum(int(np.prod(x.shape)) // c for x in shards))
    gamma = np.asarray(gamma, dtype=np.float64)
    beta = np.asarray(beta, dtype=np.float64)
    rm0 = np.zeros(c) if running is None else np.asarray(running[0], dtype=np.float64)
    rv0 = np.ones(c) if running is None else np.asarray(running[1], dtype=np.float64)
    red = lambda a: np.add.reduce(a, axis=tuple(i for i in range(a.ndim) if i != 1))  # noqa: E731
    for c0 in range(0, c, step):
        c1 = min(c, c0 + step)
        bs = (1, c1 - c0) + (1,) * (shards[0].ndim - 2)
        xb = [np.asarray(x[:, c0:c1], dtype=np.float64) for x in shards]
        s = red(xb[0])
        for x in xb[1:]:
            s = s + red(x)
        mu = s / m
        ss = None
        for x in xb:
            d = x - mu.reshape(bs)
            v = red(d * d)
            ss = v if ss is None else ss + v
        var = ss / m
        inv_std = 1.0 / np.sqrt(var + eps)
        g_, b_ = gamma[c0:c1], beta[c0:c1]
        ys, xhats, masks = [], [], []
        for x in xb:
            xh = x * inv_std.reshape(bs) + (-mu * inv_std).reshape(bs)
            y = g_.reshape(bs) * xh + b_.reshape(bs)
            mask = y > 0 if relu else None
            ys.append(y * mask if relu else y)
            xhats.append(xh)
            masks.append(mask)
        unbiased = var * (m / (m - 1.0))
        out = {"c0": c0, "c1": c1, "mu": mu, "var": var, "m": int(round(m)), "y": ys,
               "running_mean": (1.0 - momentum) * rm0[c0:c1] + momentum * mu,
               "running_var": (1.0 - momentum) * rv0[c0:c1] + momentum * unbiased}
        if dys is not None:
            gs = []
            for dy, mask in zip(dys, masks):
                gb = np.asarray(dy[:, c0:c1], dtype=np.float64)
                gs.append(gb * mask if relu else gb)
            dbeta = red(gs[0])
            dgamma = red(gs[0] * xhats[0])
            for gb, xh in zip(gs[1:], xhats[1:]):
                dbeta = dbeta + red(gb)
                dgamma = dgamma + red(gb * xh)
            a = (g_ / np.sqrt(var + eps)).reshape(bs)
            out["dx"] = [a * (gb - dbeta.reshape(bs) / m - xh * dgamma.reshape(bs) / m)
                         for gb, xh in zip(gs, xhats)]
            out["dgamma"], out["dbeta"] = dgamma, dbeta
        yield out


def rel_err(a, b, floor=1e-3):
    """Max elementwise relative error with an absolute floor on the scale — the
    reference's own comparison metric (pkg/tests/helpers.py:158-163)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return float(np.max(np.abs(a - b) / scale))
