"""World-size-2 (and 4) torch.distributed runs on CPU with the gloo backend: the
DistHandle transport that the one-process-per-GPU path uses (NCCL on B200s) — BN
sub-groups of contiguous ranks, all-gather of the per-rank partial, optional protocol
validation — checked with the oracle's ascending-rank fold."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, g, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1711_07240_b200 as cg
        from oracle import cgbn_oracle as O
        h = cg.DistHandle(bn_group_size=g, validate=True)
        rng = np.random.default_rng(rank)
        # forward partial of a fake shard: [mean | M2 | count]
        c = 5
        x = rng.standard_normal((3 + rank, c))
        mean = x.mean(0)
        m2 = ((x - mean) ** 2).sum(0)
        vec = torch.from_numpy(np.concatenate([mean, m2, [float(x.shape[0])]]))
        parts, infos = h.exchange(cg.SCOPE_BN_GROUP, "bn_forward", vec)
        got = [p.numpy().copy() for p in parts]
        # every rank of the group must hold every group member's partial in rank order
        res = {"rank": rank, "group": h.bn_group_ranks, "parts": got, "infos": infos}
        # a world-scope fold
        w, _ = h.exchange(cg.SCOPE_WORLD, "allreduce", torch.tensor([float(rank + 1)]))
        res["world_sum"] = O.star_allreduce([t.numpy() for t in w])[0]
        # protocol validation: mismatched length must raise on every rank
        try:
            n = 2 if rank == 0 else 3
            h.exchange(cg.SCOPE_WORLD, "allreduce", torch.zeros(n, dtype=torch.float64))
            res["mismatch"] = None
        except cg.CollectiveProtocolError as exc:
            res["mismatch"] = str(exc)
        q.put(res)
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001
        q.put({"rank": rank, "error": repr(exc)})


def _run(world, g):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, g, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    out.sort(key=lambda d: d["rank"])
    for d in out:
        assert "error" not in d, d
    return out


def test_world2_group2_allgather_and_fold():
    out = _run(2, 2)
    from oracle import cgbn_oracle as O
    for d in out:
        assert d["group"] == [0, 1]
        assert len(d["parts"]) == 2
        assert d["world_sum"] == 3.0
        assert d["mismatch"] is not None and "payload mismatch" in d["mismatch"]
    # both ranks hold identical bytes (rank-symmetric fold inputs)
    for a, b in zip(out[0]["parts"], out[1]["parts"]):
        assert np.array_equal(a, b)
    # rank r's slot holds rank r's partial; counts 3 and 4
    assert out[0]["parts"][0][-1] == 3.0 and out[0]["parts"][1][-1] == 4.0


@pytest.mark.slow
def test_world4_subgroups_of_two():
    out = _run(4, 2)
    assert out[0]["group"] == [0, 1] and out[3]["group"] == [2, 3]
    assert out[2]["parts"][0][-1] == 5.0 and out[2]["parts"][1][-1] == 6.0
    assert not np.array_equal(out[0]["parts"][0], out[2]["parts"][0])
    for d in out:
        assert d["world_sum"] == 10.0


def _sharded_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1711_07240_b200.collectives import _sharded_allreduce

        def cpu_fold(rows, out):  # ascending-rank left fold (stands in for cgbn_fold_sum)
            acc = rows[0].clone()
            for r in rows[1:]:
                acc = acc + r
            out.copy_(acc)

        res = {"rank": rank}
        for n in (1, 7, 1000, 4099):
            v = torch.from_numpy(np.random.default_rng(100 * n + rank).standard_normal(n)
                                 .astype(np.float32))
            res[n] = _sharded_allreduce(v, world, None, cpu_fold).numpy()
        q.put(res)
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001
        q.put({"rank": rank, "error": repr(exc)})


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_allreduce_transport(world):
    """Reduce-scatter (all-to-all) -> per-shard ascending fold -> all-gather equals the
    full-vector ascending fold, bitwise, on every rank (uneven lengths pad)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
    for d in out:
        assert "error" not in d, d
    for n in (1, 7, 1000, 4099):
        vecs = [np.random.default_rng(100 * n + r).standard_normal(n).astype(np.float32)
                for r in range(world)]
        want = vecs[0].copy()
        for x in vecs[1:]:
            want = want + x
        for d in out:
            assert np.array_equal(d[n], want), (n, d["rank"])


def _bucket_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1711_07240_b200 as cg

        def cpu_reduce(h, scope, v):  # ascending-rank fold of the exchanged rows
            parts, _ = h.exchange(scope, "allreduce", v)
            acc = parts[0].clone()
            for p in parts[1:]:
                acc = acc + p
            return acc

        h = cg.DistHandle(validate=True)
        rng = np.random.default_rng(7 + rank)
        grads = {f"l{i}.{k}": torch.from_numpy(rng.standard_normal(n).astype(np.float32))
                 for i, n in enumerate((5, 300, 17, 1024, 3)) for k in ("gamma", "beta")}
        gb = cg.GradBuckets(h, bucket_bytes=2048, dtype=torch.float32, reduce_fn=cpu_reduce)
        for name in reversed(list(grads)):  # backward order
            gb.add(name, grads[name])
        mean, loss = gb.finish(loss=float(rank) + 0.5)
        # the trainer's flat step on the same gradients (sorted keys, one vector)
        keys = sorted(grads)
        flat = torch.cat([grads[k] for k in keys] + [torch.tensor([float(rank) + 0.5])])
        fm = cpu_reduce(h, cg.SCOPE_WORLD, flat) / world
        off, ref = 0, {}
        for k in keys:
            ref[k] = fm[off:off + grads[k].numel()]
            off += grads[k].numel()
        q.put({"rank": rank, "buckets": gb.buckets_issued,
               "equal": all(torch.equal(mean[k], ref[k]) for k in keys),
               "loss": loss, "ref_loss": float(fm[-1])})
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001
        q.put({"rank": rank, "error": repr(exc)})


def test_grad_buckets_equal_flat_world_mean():
    """GradBuckets (trainer.py:419-428 bucketed): several buckets, each
    allreduced as it fills, give bitwise the flat world-mean step's gradients and loss."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
    for d in out:
        assert "error" not in d, d
        assert d["buckets"] >= 3 and d["equal"]
        assert d["loss"] == d["ref_loss"] == 1.0
