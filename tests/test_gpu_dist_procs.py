"""The N>1 path with real processes (VERDICT r1 "Next round" #5): 2 or 4 ranks, one
process each, all on GPU 0 with gloo (host-staged exchanges, so no kernel ever waits on
another process's kernel), DistHandle BN sub-groups, unequal shards, the public
sync_bn_forward / sync_bn_backward with and without ReLU, against the oracle
(oracle/cgbn_oracle.py) on the same values; plus world_mean_allreduce.

Tolerances: 1e-5 forward, 1e-4 backward (tests/test_gpu_parity.py)."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import cgbn_oracle as O

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers"))
from dist_bn_worker import shards  # noqa: E402

pytestmark = pytest.mark.gpu

WORKER = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers",
                      "dist_bn_worker.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,g", [(2, 2), (4, 2), (4, 4)])
def test_processes_match_oracle(world, g, tmp_path):
    port = str(_free_port())
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(world), str(g), port,
                               str(tmp_path)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    logs = []
    for p in procs:
        out, _ = p.communicate(timeout=300)
        logs.append(out.decode(errors="replace")[-2000:])
    assert all(p.returncode == 0 for p in procs), logs
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    xs, dys, gamma, beta = shards(world)
    for relu in (False, True):
        tag = "relu_" if relu else ""
        ref = O.cgbn_world([x.astype(np.float64) for x in xs], gamma.astype(np.float64),
                           beta.astype(np.float64), g, relu=relu,
                           dys=[d.astype(np.float64) for d in dys])
        for r in range(world):
            for key in ("y", "mu", "var", "running_mean", "running_var"):
                assert O.rel_err(got[r][tag + key], ref[r][key]) <= 1e-5, (relu, r, key)
            for key in ("dx", "dgamma", "dbeta"):
                assert O.rel_err(got[r][tag + key], ref[r][key]) <= 1e-4, (relu, r, key)
            assert int(got[r][tag + "m"]) == ref[r]["m"]
        for r in range(world):  # bitwise identical inside each BN group
            q = (r // g) * g
            for key in ("mu", "var", "dgamma", "dbeta", "running_mean"):
                assert np.array_equal(got[r][tag + key], got[q][tag + key]), (r, key)
        if g < world:  # sub-groups are isolated
            assert not np.array_equal(got[0][tag + "mu"], got[g][tag + "mu"])
    want = np.full(5, sum(range(1, world + 1)) / world)
    for r in range(world):
        assert np.array_equal(got[r]["world_mean_w"], got[0]["world_mean_w"])
        assert np.allclose(got[r]["world_mean_w"], want, rtol=0, atol=1e-15)
        assert float(got[r]["world_mean_loss"]) == sum(range(world)) / world
        assert bool(got[r]["buckets_equal"]) and int(got[r]["buckets_issued"]) >= 2
