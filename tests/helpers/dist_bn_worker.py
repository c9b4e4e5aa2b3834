"""One rank of a multi-process CGBN job on ONE GPU (tests/test_gpu_dist_procs.py).

torch.distributed with gloo (every rank on cuda:0, exchanges host-staged: two processes'
kernels never wait on each other on one GPU), DistHandle with BN sub-groups, the public
sync_bn_forward / sync_bn_backward on this rank's shard. The shards are generated from
one seed by every rank, so the parent can run the oracle on the same values. Results go
to <out>/rank<r>.npz.

    python tests/helpers/dist_bn_worker.py RANK WORLD G PORT OUTDIR
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def shards(world, seed=11):
    """Unequal per-rank batches (the reference allows them)."""
    rng = np.random.default_rng(seed)
    batches = [2 + (r % 3) for r in range(world)]
    c, h, w = 24, 7, 9
    xs = [(1.5 + rng.standard_normal((b, c, h, w))).astype(np.float32) for b in batches]
    dys = [rng.standard_normal((b, c, h, w)).astype(np.float32) for b in batches]
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.standard_normal(c).astype(np.float32)
    return xs, dys, gamma, beta


def main():
    rank, world, g, port, out = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]),
                                 sys.argv[4], sys.argv[5])
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port, RANK=str(rank),
                      WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1711_07240_b200 as cg
    dev = torch.device("cuda", 0)
    h = cg.DistHandle(bn_group_size=g, device=dev, validate=True)
    xs, dys, gamma, beta = shards(world)
    res = {}
    for relu in (False, True):
        st = cg.BNLayerState(gamma=gamma, beta=beta)
        x = torch.from_numpy(xs[rank]).to(dev)
        y, cache = cg.sync_bn_forward(h, x, st, relu=relu)
        dx, dg, db = cg.sync_bn_backward(h, torch.from_numpy(dys[rank]).to(dev), cache, st)
        tag = "relu_" if relu else ""
        res.update({tag + "y": y.cpu().numpy(), tag + "dx": dx.cpu().numpy(),
                    tag + "mu": cache.mu.cpu().numpy(), tag + "var": cache.var.cpu().numpy(),
                    tag + "running_mean": st.running_mean.cpu().numpy(),
                    tag + "running_var": st.running_var.cpu().numpy(),
                    tag + "dgamma": dg.cpu().numpy(), tag + "dbeta": db.cpu().numpy(),
                    tag + "m": np.array(cache.total_count)})
    # the trainer's world gradient step over the same job (trainer.py:419-428)
    grads = {"w": torch.full((5,), float(rank + 1), device=dev, dtype=torch.float64)}
    mean, loss = cg.world_mean_allreduce(h, grads, loss=float(rank))
    res["world_mean_w"] = mean["w"].cpu().numpy()
    res["world_mean_loss"] = np.array(loss)
    # the same step bucketed and overlapped on a side stream (GradBuckets)
    more = {f"g{i}": torch.randn(40 + i, device=dev, dtype=torch.float64,
                                 generator=torch.Generator(device=dev).manual_seed(rank * 10 + i))
            for i in range(6)}
    more["w"] = grads["w"]
    flat_mean, flat_loss = cg.world_mean_allreduce(h, more, loss=float(rank))
    gb = cg.GradBuckets(h, bucket_bytes=512, dtype=torch.float64)
    for k in reversed(sorted(more)):
        gb.add(k, more[k])
    bmean, bloss = gb.finish(loss=float(rank))
    res["buckets_issued"] = np.array(gb.buckets_issued)
    res["buckets_equal"] = np.array(all(torch.equal(bmean[k], flat_mean[k]) for k in more)
                                    and bloss == flat_loss)
    np.savez(os.path.join(out, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
