"""Host-side logic on CPU: the threaded DeviceGroup transport (rendezvous, sequence and
payload checks, timeouts, abort fan-out — collectives.py:98-298 semantics), the
BN-group topology, and that the product path refuses CPU tensors (no fallback)."""

import threading

import numpy as np
import pytest
import torch

import paper_1711_07240_b200 as cg
from paper_1711_07240_b200.collectives import SoloHandle
from paper_1711_07240_b200.tensor import TensorError, geometry
from oracle import cgbn_oracle as O


def cpu_group(world, g=None, timeout=5.0):
    return cg.DeviceGroup(world, bn_group_size=g, timeout_s=timeout,
                          devices=["cpu"] * world)


def test_group_topology():
    grp = cpu_group(6, 3)
    h = grp.handles
    assert [x.bn_group_index for x in h] == [0, 0, 0, 1, 1, 1]
    assert h[4].bn_group_ranks == [3, 4, 5]
    with pytest.raises(ValueError):
        cg.DeviceGroup(4, bn_group_size=3, devices=["cpu"] * 4)
    with pytest.raises(ValueError):
        cg.DeviceGroup(0)


def test_exchange_returns_rank_order_and_infos():
    grp = cpu_group(4, 2)

    def fn(h):
        v = torch.full((3,), float(h.rank + 1), dtype=torch.float64)
        parts, infos = h.exchange(cg.SCOPE_BN_GROUP, "probe", v, info=10 * h.rank)
        return [p.tolist() for p in parts], infos

    out = grp.run(fn)
    assert out[0][0] == [[1.0] * 3, [2.0] * 3] and out[0][1] == [0, 10]
    assert out[3][0] == [[3.0] * 3, [4.0] * 3] and out[3][1] == [20, 30]


def test_bn_group_fold_equals_oracle_star_allreduce():
    # transport + ascending fold (oracle as the checker) == reference allreduce_sum
    grp = cpu_group(4, 4)
    rng = np.random.default_rng(0)
    vecs = [rng.standard_normal(5) for _ in range(4)]

    def fn(h):
        parts, _ = h.exchange(cg.SCOPE_WORLD, "probe", torch.from_numpy(vecs[h.rank]))
        return O.star_allreduce([p.numpy() for p in parts])

    out = grp.run(fn)
    want = O.star_allreduce(vecs)
    for o in out:
        assert np.array_equal(o, want)


def test_payload_mismatch_names_ranks():
    grp = cpu_group(2)

    def fn(h):
        n = 3 if h.rank == 0 else 4
        return h.exchange(cg.SCOPE_WORLD, "allreduce", torch.zeros(n, dtype=torch.float64))

    with pytest.raises(cg.CollectiveProtocolError, match="rank 0: len 3.*rank 1: len 4"):
        grp.run(fn)


def test_kind_mismatch():
    grp = cpu_group(2)

    def fn(h):
        kind = "bn_forward" if h.rank == 0 else "bn_backward"
        return h.exchange(cg.SCOPE_WORLD, kind, torch.zeros(2, dtype=torch.float64))

    with pytest.raises(cg.CollectiveProtocolError, match="different"):
        grp.run(fn)


def test_timeout_names_missing_rank():
    grp = cpu_group(2, timeout=0.5)

    def fn(h):
        if h.rank == 1:
            return None  # never joins
        return h.exchange(cg.SCOPE_WORLD, "allreduce", torch.zeros(2, dtype=torch.float64))

    with pytest.raises(cg.CollectiveTimeoutError, match=r"\[1\]"):
        grp.run(fn)


def test_worker_death_aborts_peers_quickly():
    grp = cpu_group(3, timeout=30.0)

    def fn(h):
        if h.rank == 2:
            raise RuntimeError("boom")
        return h.exchange(cg.SCOPE_WORLD, "allreduce", torch.zeros(2, dtype=torch.float64))

    import time
    t0 = time.monotonic()
    with pytest.raises(RuntimeError, match="boom"):
        grp.run(fn)
    assert time.monotonic() - t0 < 5.0


def test_sequence_numbers_keep_scopes_apart():
    grp = cpu_group(4, 2)

    def fn(h):
        outs = []
        for i in range(5):
            v = torch.tensor([float(h.rank * 10 + i)], dtype=torch.float64)
            p, _ = h.exchange(cg.SCOPE_BN_GROUP, "bn", v)
            q, _ = h.exchange(cg.SCOPE_WORLD, "w", v)
            outs.append((sum(x.item() for x in p), sum(x.item() for x in q)))
        return outs

    out = grp.run(fn)
    for i in range(5):
        assert out[0][i][0] == out[1][i][0] == 0 + 10 + 2 * i
        assert out[2][i][0] == out[3][i][0] == 20 + 30 + 2 * i
        assert all(out[r][i][1] == 60 + 4 * i for r in range(4))


def test_sequence_skew_diagnosed():
    """A rank whose sequence number runs ahead (a skipped or extra collective) is
    diagnosed, not paired with the wrong call (test_collectives.py:216-227)."""
    grp = cpu_group(2, timeout=2.0)

    def fn(h):
        if h.rank == 1:
            h._next_seq("world")  # simulates a skipped / extra call
        return h.exchange(cg.SCOPE_WORLD, "allreduce", torch.ones(1, dtype=torch.float64))

    with pytest.raises(cg.CollectiveError, match="#"):
        grp.run(fn)


def test_return_exceptions():
    grp = cpu_group(2)

    def fn(h):
        if h.rank == 0:
            raise ValueError("x")
        return 7

    out = grp.run(fn, return_exceptions=True)
    assert isinstance(out[0], ValueError) and out[1] == 7


def test_solo_handle_identity_exchange():
    h = SoloHandle(device="cpu")
    v = torch.arange(3.0)
    parts, infos = h.exchange(cg.SCOPE_BN_GROUP, "bn", v, info=5)
    assert parts[0] is v and infos == [5]
    with pytest.raises(cg.CollectiveProtocolError):
        h.exchange("nope", "bn", v)


def test_product_path_refuses_cpu_tensors():
    with pytest.raises(TensorError, match="no CPU fallback"):
        geometry(torch.zeros(2, 3))
    with pytest.raises(TensorError):
        geometry(torch.zeros(2, 3, 4))
    h = SoloHandle(device="cpu")
    with pytest.raises(cg.CollectiveProtocolError, match="CUDA"):
        cg.allreduce_sum(h, cg.SCOPE_WORLD, torch.zeros(3))


def test_set_forward_exchange_modes():
    prev = cg.set_forward_exchange("reference")
    assert cg.set_forward_exchange(prev) == "reference"
    with pytest.raises(ValueError):
        cg.set_forward_exchange("two_pass")
