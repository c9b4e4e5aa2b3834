"""Generate the golden parity fixtures by running the REAL reference.

Imports ``bigbatch`` from /root/reference/pkg/src (read-only; never copied) and runs its
stock CGBN path — ``DeviceGroup(world, bn_group_size).run`` with ``sync_bn_forward`` /
``sync_bn_backward`` exactly as its own tests do (test_batchnorm.py:31-40,
test_acceptance.py:73-80) — on seeded float32 inputs (passed to the reference as the
same values in float64, its default dtype). Writes one ``<case>.npz`` per case next to
this script. Run in the build container (the GPU box has no /root/reference):

    python tests/golden/make_golden.py
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import bigbatch  # noqa: E402
from bigbatch import (BNLayerState, DeviceGroup, Tensor, bn_forward_local,  # noqa: E402
                      sync_bn_backward, sync_bn_forward)

HERE = os.path.dirname(os.path.abspath(__file__))

# name: (world, bn_group, per-rank shapes, loc, scale, one_pass, relu, momentum, eps, init_running)
CASES = {
    "config1_mini": (4, 4, [(2, 8, 7, 9)] * 4, 0.0, 1.0, False, False, 0.1, 1e-5, False),
    "unequal_shards": (3, 3, [(1, 5, 4, 4), (3, 5, 4, 4), (2, 5, 4, 4)], 0.0, 1.0, False, False, 0.1, 1e-5, False),
    "subgroups": (4, 2, [(2, 3, 5, 5), (1, 3, 5, 5), (3, 3, 5, 5), (2, 3, 5, 5)], 0.0, 1.0, False, False, 0.1, 1e-5, False),
    "one_pass_loc2": (3, 3, [(3, 4, 2, 2)] * 3, 2.0, 1.0, True, False, 0.1, 1e-5, False),
    "cancellation_loc100": (2, 2, [(4, 6, 8, 8)] * 2, 100.0, 1.0, False, False, 0.1, 1e-5, False),
    "two_d": (2, 2, [(5, 6), (3, 6)], 0.0, 1.0, False, False, 0.1, 1e-5, False),
    "hw49": (2, 2, [(2, 16, 7, 7)] * 2, 0.0, 1.0, False, False, 0.1, 1e-5, False),
    "hw_odd_1050": (2, 2, [(1, 4, 25, 42)] * 2, 0.5, 2.0, False, False, 0.1, 1e-5, False),
    "relu": (2, 2, [(2, 6, 6, 6)] * 2, 0.0, 1.0, False, True, 0.1, 1e-5, False),
    "group_of_one": (2, 1, [(3, 4, 3, 3), (2, 4, 3, 3)], 0.0, 1.0, False, False, 0.1, 1e-5, False),
    "momentum_running": (2, 2, [(2, 5, 4, 6)] * 2, -1.0, 3.0, False, False, 0.25, 1e-3, True),
    "single_rank_large_c": (1, 1, [(2, 64, 3, 3)], 0.0, 1.0, False, False, 0.1, 1e-5, False),
}


def make_case(name, world, g, shapes, loc, scale, one_pass, relu, momentum, eps, init_running):
    rng = np.random.default_rng([ord(ch) for ch in name])
    c = shapes[0][1]
    xs = [(loc + scale * rng.standard_normal(s)).astype(np.float32) for s in shapes]
    dys = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.standard_normal(c).astype(np.float32)
    if init_running:
        rm0 = rng.standard_normal(c).astype(np.float32)
        rv0 = rng.uniform(0.5, 2.0, c).astype(np.float32)
    else:
        rm0 = np.zeros(c, np.float32)
        rv0 = np.ones(c, np.float32)

    def mk():
        return BNLayerState(gamma=gamma.astype(np.float64), beta=beta.astype(np.float64),
                            eps=eps, running_mean=rm0.astype(np.float64),
                            running_var=rv0.astype(np.float64), running_momentum=momentum)

    def worker(h):
        st = mk()
        y, cache = sync_bn_forward(h, Tensor(xs[h.rank].astype(np.float64)), st,
                                   one_pass=one_pass)
        yv = y.array
        dy = dys[h.rank].astype(np.float64)
        if relu:  # the reference model's relu layer after bn (model.py:243-246, 330-331)
            mask = yv > 0
            yv = yv * mask
            dy = dy * mask
        dx, dgamma, dbeta = sync_bn_backward(h, Tensor(dy), cache, st)
        return dict(y=yv, mu=cache.mu, var=cache.var, m=cache.total_count,
                    running_mean=st.running_mean, running_var=st.running_var,
                    dx=dx.array, dgamma=dgamma, dbeta=dbeta, x_hat=cache.x_hat.array)

    outs = DeviceGroup(world, bn_group_size=g, timeout_s=60.0).run(worker)
    arrays = dict(gamma=gamma, beta=beta, running_mean0=rm0, running_var0=rv0)
    for r in range(world):
        arrays[f"x_{r}"] = xs[r]
        arrays[f"dy_{r}"] = dys[r]
        for k, v in outs[r].items():
            arrays[f"{k}_{r}"] = np.asarray(v)
    # eval-mode output of rank 0's shard under the post-update running stats of rank 0
    st = BNLayerState(gamma=gamma.astype(np.float64), beta=beta.astype(np.float64), eps=eps,
                      running_mean=outs[0]["running_mean"].astype(np.float32).astype(np.float64),
                      running_var=outs[0]["running_var"].astype(np.float32).astype(np.float64),
                      running_momentum=momentum)
    yev, _ = bn_forward_local(Tensor(xs[0].astype(np.float64)), st, mode="eval")
    arrays["eval_y_0"] = yev.array
    meta = dict(name=name, world=world, bn_group=g, shapes=[list(s) for s in shapes],
                loc=loc, scale=scale, one_pass=one_pass, relu=relu, momentum=momentum,
                eps=eps, reference=f"bigbatch {bigbatch.__version__}")
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)


if __name__ == "__main__":
    for name, spec in CASES.items():
        make_case(name, *spec)
        print("wrote", name)
