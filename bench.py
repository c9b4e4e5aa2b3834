#!/usr/bin/env python3
"""CGBN forward+backward benchmark (BASELINE.json metric, configs[1]).

Workload ("resnet50_bn_b32"): every BatchNorm layer of ResNet-50 (53 layers, C=64..2048,
224x224 input) at batch 32 per GPU, fp32 NCHW. One step = the CGBN forward of all 53
layers followed by their CGBN backward in reverse order — per layer: stats kernel ->
statistics exchange over the BN group (= all N GPUs, NCCL all-gather; identity at N=1)
-> normalise (+running-stat update) kernel; backward reduce kernel -> exchange -> dx
kernel. Weak scaling: every GPU holds its own batch of 32.

metric value = algorithmic bytes (32 B per fp32 activation element: fwd 12, bwd 20,
SURVEY.md §8d) of the whole job / device time per step, max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cgbn|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CGBN fwd+bwd algorithmic GB/s (whole job; per-GPU and % HBM roofline in extra keys)"
UNIT = "GB/s"
BYTES_PER_ELEM = 32  # fwd 12 + bwd 20


L2_BYTES = 126 * 1024 * 1024


def _cdiv(a, b):
    return -(-a // b)


def resnet50_bn_shapes(batch=32, h=224, w=None):
    """The 53 BN layers of torchvision ResNet-50 (v1.5: stride on conv2); feature maps
    are ceil(input / stride) (224x224 -> 112, 56, 28, 14, 7)."""
    w = h if w is None else w
    sh, sw = _cdiv(h, 2), _cdiv(w, 2)
    shapes = [(batch, 64, sh, sw)]  # stem bn1
    res = [(_cdiv(h, s), _cdiv(w, s)) for s in (4, 8, 16, 32)]
    cfg = [(64, 256, 3, res[0], res[0]), (128, 512, 4, res[0], res[1]),
           (256, 1024, 6, res[1], res[2]), (512, 2048, 3, res[2], res[3])]
    for width, out, blocks, in_hw, hw in cfg:
        for b in range(blocks):
            h1 = in_hw if b == 0 else hw
            shapes.append((batch, width) + h1)   # bn1 (after 1x1 conv, input res)
            shapes.append((batch, width) + hw)   # bn2 (after strided 3x3)
            shapes.append((batch, out) + hw)     # bn3
            if b == 0:
                shapes.append((batch, out) + hw)  # downsample bn
    return shapes


def fpn_neck_shapes(batch=2, h=800, w=1333, c=256):
    """One BN per FPN level P2..P6 at 800x1333."""
    return [(batch, c, _cdiv(h, s), _cdiv(w, s)) for s in (4, 8, 16, 32, 64)]


# SURVEY.md 8(d) configurations. The default (what the driver runs) is config 2.
WORKLOADS = {
    "resnet50_bn_b32": ("config 2: ResNet-50 BN layers, 32 images/GPU at 224x224",
                        lambda: resnet50_bn_shapes(32)),
    "fpn_neck_800x1333": ("config 3: FPN neck BN (C=256, P2..P6), 2 images/GPU at 800x1333",
                          lambda: fpn_neck_shapes(2)),
    "megdet_r50fpn_800x1333": ("config 4: MegDet R50 backbone + FPN neck BN, 2 images/GPU "
                               "at 800x1333", lambda: resnet50_bn_shapes(2, 800, 1333)
                               + fpn_neck_shapes(2)),
    "latency_2048x7x7": ("config 5: one latency-bound layer [1,2048,7,7]",
                         lambda: [(1, 2048, 7, 7)]),
}


def host_cpu_info():
    """CPU model, os.cpu_count() and the affinity mask size (SURVEY 8(d) asks for all)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        aff = None
    return {"cpu_model": model, "host_cpus": os.cpu_count(), "affinity_cpus": aff}


def _lib_consts():
    """The C ABI's layout / dtype codes (include/cgbn.h via the binding module)."""
    from paper_1711_07240_b200 import _lib
    return _lib


def numel(s):
    n = 1
    for e in s:
        n *= e
    return n


# ----------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"cgbn_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------------
# reference arm / CPU baseline (the reference's own CPU implementation)

def _reference_module():
    """The UNMODIFIED reference (bigbatch) installed in baseline/_ref, else None."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "bigbatch")):
        sys.path.insert(0, ref_dir)
        try:
            import bigbatch  # noqa: F401
            return bigbatch
        except Exception:  # noqa: BLE001
            return None
    return None


def reference_step(bb, shape, ranks, seed):
    """One CGBN fwd+bwd of one layer through the reference's stock path:
    DeviceGroup(ranks).run with sync_bn_forward + sync_bn_backward (f64, its default).
    Returns (seconds, algorithmic bytes)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    xs = [rng.standard_normal(shape).astype(np.float32).astype(np.float64) for _ in range(ranks)]
    dys = [rng.standard_normal(shape).astype(np.float32).astype(np.float64) for _ in range(ranks)]
    c = shape[1]
    gamma = rng.uniform(0.5, 1.5, c)
    beta = rng.standard_normal(c)
    t_in = [bb.Tensor(x) for x in xs]
    d_in = [bb.Tensor(d) for d in dys]

    def worker(h):
        st = bb.BNLayerState(gamma=gamma.copy(), beta=beta.copy())
        _, cache = bb.sync_bn_forward(h, t_in[h.rank], st)
        bb.sync_bn_backward(h, d_in[h.rank], cache, st)

    g = bb.DeviceGroup(ranks)
    t0 = time.perf_counter()
    g.run(worker)
    return time.perf_counter() - t0, BYTES_PER_ELEM * numel(shape) * ranks


def port_step(shape, ranks, seed):
    """Fallback when baseline/_ref is absent: the oracle port (oracle/cgbn_oracle.py)."""
    import numpy as np
    from oracle import cgbn_oracle as O
    rng = np.random.default_rng(seed)
    xs = [rng.standard_normal(shape).astype(np.float32).astype(np.float64) for _ in range(ranks)]
    dys = [rng.standard_normal(shape).astype(np.float32).astype(np.float64) for _ in range(ranks)]
    c = shape[1]
    t0 = time.perf_counter()
    O.cgbn_world(xs, rng.uniform(0.5, 1.5, c), rng.standard_normal(c), ranks, dys=dys)
    return time.perf_counter() - t0, BYTES_PER_ELEM * numel(shape) * ranks


def cpu_sample(shapes, ranks, budget_s, max_units=None, min_units=1, start=0):
    """Run the workload's layers at their own shapes (the config's batch per rank),
    cycling from layer `start`, through the reference until budget_s elapsed. Returns
    dict."""
    bb = _reference_module()
    kind = "reference" if bb is not None else "port"
    t_total, b_total, units = 0.0, 0, 0
    i = start
    while True:
        shape = tuple(shapes[i % len(shapes)])
        dt, nb = (reference_step(bb, shape, ranks, i) if bb is not None
                  else port_step(shape, ranks, i))
        t_total += dt
        b_total += nb
        units += 1
        i += 1
        if max_units is not None and units >= max_units:
            break
        if units >= min_units and t_total >= budget_s:
            break
    return {"kind": kind, "seconds": t_total, "bytes": b_total, "units": units,
            "gbs": b_total / t_total / 1e9}


def _ref_proc(q, barrier, workload, n, steps, warmup, offset):
    """One reference worker process: warm up, wait for the others, time `steps`
    layer-steps (reference_step's own timer: the stock sync_bn_forward+backward)."""
    bb = _reference_module()
    shapes = WORKLOADS[workload][1]()

    def one(k):
        shape = tuple(shapes[k % len(shapes)])  # the config's own layer shape (batch 32)
        return reference_step(bb, shape, n, k) if bb is not None else port_step(shape, n, k)

    for i in range(warmup):
        one(offset + i)
    barrier.wait()
    t_total, b_total = 0.0, 0
    for k in range(steps):
        dt, nb = one(offset + k)
        t_total += dt
        b_total += nb
    q.put((t_total, b_total))


def reference_procs(shapes, n, requested=None):
    """Worker processes for the reference arm: one per allowed core (the reference is
    GIL-bound NumPy, so threads do not add throughput), capped by available memory."""
    try:
        cores = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        cores = os.cpu_count() or 1
    procs = cores if requested is None else max(1, min(requested, cores))
    try:
        import psutil
        avail = psutil.virtual_memory().available
        peak = max(numel(s) for s in shapes) * 8 * n * 16  # f64 copies of the largest layer
        procs = max(1, min(procs, int(0.5 * avail // max(peak, 1))))
    except Exception:  # noqa: BLE001
        pass
    return procs


def run_reference_arm(args):
    import multiprocessing as mp
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = args.gpus
    shapes = WORKLOADS[args.workload][1]()
    bb = _reference_module()
    kind = "reference" if bb is not None else "port"
    procs = reference_procs(shapes, n, args.ref_procs)
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    barrier = ctx.Barrier(procs)
    # process p starts at layer p * len(shapes) / procs, so together they cover the
    # workload's layers (with the config's own shapes) rather than one corner of it
    ps = [ctx.Process(target=_ref_proc,
                      args=(q, barrier, args.workload, n, args.steps, min(args.warmup, 1),
                            (p * len(shapes)) // procs))
          for p in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    t_max = max(t for t, _ in res)
    b_total = sum(b for _, b in res)
    value = b_total / t_max / 1e9
    sample = (f"{procs} concurrent processes x {args.steps} layer-steps each; a step is one "
              f"{args.workload} BN layer at its own shape (batch {shapes[0][0]} per simulated "
              f"device, the GPU arm's shapes; the processes start at evenly spaced layers and "
              f"cycle through the {len(shapes)}), {n} device(s) as the reference's DeviceGroup "
              f"threads, f64 (reference default), stock sync_bn_forward+sync_bn_backward; value "
              f"= all processes' bytes / the slowest process's time")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": args.workload, "describe": WORKLOADS[args.workload][0],
                   "per_gpu_batch": shapes[0][0], "layers_sampled": min(len(shapes),
                                                                         procs * args.steps),
                   "parallelism": f"cgbn_group{n}", "bn_group_size": n, "layout": "NCHW"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": kind,
                         "sample": sample, **host_cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------------
# GPU arm

def _layer_paths(lib, shapes, lay):
    """Which layers the single-rank step runs on chip (one kernel per direction,
    cgbn_onchip.cuh) and which on the split kernels."""
    fwd, bwd = [], []
    for s in shapes:
        n, c, h, w = s
        fwd.append(bool(lib.cgbn_onchip_selected(n, c, h * w, lay, 0)))
        bwd.append(bool(lib.cgbn_onchip_selected(n, c, h * w, lay, 1)))
    return fwd, bwd


# Bytes per element each kernel family must move: the split passes'
# algorithmic traffic, and the on-chip passes' compulsory traffic (the activation is read
# once and held on chip across the statistics). The bench metric keeps 32 B/elem.
FAMILY_BPE = {"fwd_onchip": 8, "bwd_onchip": 12, "fwd_stats": 4, "fwd_normalize": 8,
              "bwd_reduce": 8, "bwd_dx": 12}


def _traffic_for(family, layout="nchw", act="f32"):
    """ncu dram bytes per launch of a kernel family from the committed launch-list
    summary (profiles/r2_traffic*.json, regenerated by tools/step_breakdown.py --traffic);
    (None, reason) when the file or the family is absent."""
    name = "r2_traffic.json" if (layout, act) == ("nchw", "f32") else \
        f"r2_traffic_{layout}_{act}.json"
    path = os.path.join(ROOT, "profiles", name)
    try:
        fams = json.load(open(path))["families"]
        return fams[family]["dram_bytes_per_launch"], f"profiles/{name}"
    except Exception:  # noqa: BLE001
        return None, f"profiles/{name} has no '{family}'"


def kernel_profile(cg, shapes, xs, dys, states, handle, reps=20, lay=0, esize=4):
    """Per-family device time of the step's kernels, each family timed DIRECTLY: a CUDA
    graph holds that family's launch for every layer it serves (the layers' own buffers,
    step order: forward families in layer order, backward ones reversed), made through
    the C ABI; CUDA events on the replay stream around `reps` replays.

    Families: the single-launch on-chip passes (cgbn_fwd_train_local / cgbn_bwd_local on
    the layers that fit on chip) and, for the other layers, the split kernels --
    statistics (cgbn_fwd_stats), normalise (cgbn_fwd_normalize on the rank's own partial:
    finalize + elementwise pass), backward reduce (cgbn_bwd_reduce) and dx
    (cgbn_bwd_dx). A family graph runs one family's kernels back to back, so a pass
    finds nothing of its layer in L2 from the pass before it (unlike inside the step):
    these are L2-cold per-kernel times, the step time is the in-context total.
    Returns ({family: stats}, description)."""
    import torch
    from paper_1711_07240_b200 import _lib
    from paper_1711_07240_b200.tensor import workspace
    lib = _lib.load()
    dev = xs[0].device
    on_f, on_b = _layer_paths(lib, shapes, lay)
    # one eager forward to obtain every layer's saved statistics
    caches = [cg.sync_bn_forward(handle, x, st)[1] for x, st in zip(xs, states)]
    torch.cuda.synchronize()
    side = torch.cuda.Stream(device=dev)
    L = []
    for k, (s, x, dy, st, ca) in enumerate(zip(shapes, xs, dys, states, caches)):
        n, c, h, w = s
        part = torch.empty(2 * c + 1, dtype=torch.float64, device=dev)
        bpart = torch.empty(2 * c, dtype=torch.float64, device=dev)
        pa, ka = _lib.ptr_array([part.data_ptr()])
        pb, kb = _lib.ptr_array([bpart.data_ptr()])
        L.append(dict(k=k, n=n, c=c, hw=h * w, x=x, dy=dy, st=st, saved=ca.saved,
                      y=torch.empty_like(x), dx=torch.empty_like(x), part=part, bpart=bpart,
                      pa=pa, pb=pb, keep=(ka, kb),
                      dg=torch.empty(c, device=dev), db=torch.empty(c, device=dev),
                      rm=torch.zeros(c, device=dev), rv=torch.ones(c, device=dev),
                      saved2=torch.empty(3 * c + 1, dtype=torch.float64, device=dev),
                      status=torch.zeros(1, dtype=torch.int32, device=dev)))
    fwd_local = lambda d, ws, st: lib.cgbn_fwd_train_local(  # noqa: E731
        d["x"].data_ptr(), d["n"], d["c"], d["hw"], lay, d["st"].gamma.data_ptr(),
        d["st"].beta.data_ptr(), 1e-5, 0.1, d["rm"].data_ptr(), d["rv"].data_ptr(),
        d["saved2"].data_ptr(), 0, d["y"].data_ptr(), d["status"].data_ptr(),
        ws.data_ptr(), ws.numel(), st)
    bwd_local = lambda d, ws, st: lib.cgbn_bwd_local(  # noqa: E731
        d["dy"].data_ptr(), d["x"].data_ptr(), d["n"], d["c"], d["hw"], lay,
        d["saved"].data_ptr(), d["st"].gamma.data_ptr(), d["st"].beta.data_ptr(), 1e-5,
        0, d["dx"].data_ptr(), d["dg"].data_ptr(), d["db"].data_ptr(),
        d["status"].data_ptr(), ws.data_ptr(), ws.numel(), st)
    fams = {
        "fwd_onchip": ([d for d in L if on_f[d["k"]]], fwd_local),
        "fwd_stats": ([d for d in L if not on_f[d["k"]]], lambda d, ws, st: lib.cgbn_fwd_stats(
            d["x"].data_ptr(), d["n"], d["c"], d["hw"], lay, d["part"].data_ptr(),
            ws.data_ptr(), ws.numel(), st)),
        "fwd_normalize": ([d for d in L if not on_f[d["k"]]],
                          lambda d, ws, st: lib.cgbn_fwd_normalize(
            d["x"].data_ptr(), d["n"], d["c"], d["hw"], lay, d["pa"], 1,
            d["st"].gamma.data_ptr(), d["st"].beta.data_ptr(), 1e-5, 0.1, d["rm"].data_ptr(),
            d["rv"].data_ptr(), d["saved2"].data_ptr(), 0, d["y"].data_ptr(),
            d["status"].data_ptr(), ws.data_ptr(), ws.numel(), st)),
        "bwd_onchip": ([d for d in reversed(L) if on_b[d["k"]]], bwd_local),
        "bwd_reduce": ([d for d in reversed(L) if not on_b[d["k"]]],
                       lambda d, ws, st: lib.cgbn_bwd_reduce(
            d["dy"].data_ptr(), d["x"].data_ptr(), d["n"], d["c"], d["hw"], lay,
            d["saved"].data_ptr(), d["st"].gamma.data_ptr(), d["st"].beta.data_ptr(), 0,
            d["bpart"].data_ptr(), ws.data_ptr(), ws.numel(), st)),
        "bwd_dx": ([d for d in reversed(L) if not on_b[d["k"]]],
                   lambda d, ws, st: lib.cgbn_bwd_dx(
            d["dy"].data_ptr(), d["x"].data_ptr(), d["n"], d["c"], d["hw"], lay, d["pb"], 1,
            d["saved"].data_ptr(), d["st"].gamma.data_ptr(), d["st"].beta.data_ptr(), 1e-5, 0,
            d["dx"].data_ptr(), d["dg"].data_ptr(), d["db"].data_ptr(), d["status"].data_ptr(),
            ws.data_ptr(), ws.numel(), st)),
    }
    out = {}
    with torch.cuda.stream(side):
        ws = workspace(dev, max(lib.cgbn_workspace_bytes(d["n"], d["c"], d["hw"], lay) for d in L))
        st = side.cuda_stream
        # the partials the normalise / dx families consume (their own rank's, G = 1)
        for d in L:
            _lib.check(fams["fwd_stats"][1](d, ws, st), "fwd_stats")
            _lib.check(fams["bwd_reduce"][1](d, ws, st), "bwd_reduce")
        for name, (layers, fn) in fams.items():
            if not layers:
                continue
            for d in layers:
                _lib.check(fn(d, ws, st), name)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for d in layers:
                    fn(d, ws, side.cuda_stream)
            g.replay()
            side.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(side)
            for _ in range(reps):
                g.replay()
            e1.record(side)
            side.synchronize()
            ms = e0.elapsed_time(e1) / reps
            del g
            bpe = FAMILY_BPE[name] * esize // 4  # bytes scale with the activation size
            elems = sum(d["n"] * d["c"] * d["hw"] for d in layers)
            out[name] = {"ms_per_step": ms, "launches_per_step": len(layers),
                         "bytes_per_elem": bpe, "elements": elems,
                         "alg_bytes_per_launch": bpe * elems / len(layers),
                         "alg_gbs": bpe * elems / (ms * 1e-3) / 1e9}
    tot = sum(v["ms_per_step"] for v in out.values())
    for v in out.values():
        v["share"] = v["ms_per_step"] / tot
    return out, ("each family timed directly: one CUDA graph of that family's launches over "
                 "the step's layers (layer buffers, step order) through the C ABI, CUDA "
                 f"events on the replay stream, mean of {reps} replays; L2-cold per kernel")


def bench_parity(cg, torch, shapes, xs, dys, states, dev, esize):
    """After timing: the public API on three of the step's own layers (the largest, a 7x7
    and a 28x28 one, their timed input buffers) against the f64 oracle (the reference's
    two-pass arithmetic, batchnorm.py:115-252; oracle/ is the checker, not the measured
    path). Tolerances as in tests/: 1e-5 forward, 1e-4 backward (fp32 activations); 16-bit
    activations add their output rounding (y, dx: 1e-2)."""
    import numpy as np
    from oracle import cgbn_oracle as O
    pick = [max(range(len(shapes)), key=lambda i: numel(shapes[i]))]
    for hw in (7, 28):
        cand = [i for i, s in enumerate(shapes) if s[2] == hw and i not in pick]
        if cand:
            pick.append(max(cand, key=lambda i: numel(shapes[i])))
    # 16-bit activations: y and dx carry one rounding to the activation dtype
    # (tests/test_gpu_half.py OUT_TOL)
    if esize == 4:
        tol_y, tol_dx = 1e-5, 1e-4
    else:
        tol_y = tol_dx = 8e-3 if xs[0].dtype == torch.bfloat16 else 1.5e-3
    worst = {}
    layers = []
    h = cg.SoloHandle(dev)
    for i in pick:
        g0, b0 = states[i].gamma.detach().clone(), states[i].beta.detach().clone()
        st = cg.BNLayerState(gamma=g0, beta=b0)
        y, cache = cg.sync_bn_forward(h, xs[i], st)
        dx, dg, db = cg.sync_bn_backward(h, dys[i], cache, st)
        torch.cuda.synchronize()
        xh = xs[i].float().cpu().numpy()
        dyh = dys[i].float().cpu().numpy()
        got = {"y": y.float().cpu().numpy(), "dx": dx.float().cpu().numpy(),
               "mu": cache.mu.cpu().numpy(), "var": cache.var.cpu().numpy(),
               "running_mean": st.running_mean.cpu().numpy(),
               "running_var": st.running_var.cpu().numpy(),
               "dgamma": dg.cpu().numpy(), "dbeta": db.cpu().numpy()}
        err = {k: 0.0 for k in got}
        for b in O.group_blocks([xh], g0.cpu().numpy(), b0.cpu().numpy(), dys=[dyh]):
            c0, c1 = b["c0"], b["c1"]
            err["y"] = max(err["y"], O.rel_err(got["y"][:, c0:c1], b["y"][0]))
            err["dx"] = max(err["dx"], O.rel_err(got["dx"][:, c0:c1], b["dx"][0]))
            for k in ("mu", "var", "running_mean", "running_var", "dgamma", "dbeta"):
                err[k] = max(err[k], O.rel_err(got[k][c0:c1], b[k]))
        layers.append({"layer": i, "shape": list(shapes[i]), "max_rel_err": err})
        for k, v in err.items():
            worst[k] = max(worst.get(k, 0.0), v)
        del y, dx, cache, got
    tol = {"y": tol_y, "mu": 1e-5, "var": 1e-5, "running_mean": 1e-5, "running_var": 1e-5,
           "dx": tol_dx, "dgamma": 1e-4, "dbeta": 1e-4}
    return {"layers": layers, "max_rel_err": worst, "tol": tol,
            "ok": all(worst[k] <= tol[k] for k in worst),
            "how": "sync_bn_forward/sync_bn_backward (group of one) on the timed layers' own "
                   "x / dy after the timed region, vs oracle.cgbn_oracle.group_blocks (f64); "
                   "rel_err = max|a-b| / max(|a|, |b|, 1e-3) (helpers.py:158-163)"}


def count_graph_kernels(graph):
    """Kernel nodes of a captured step (cuda-python on the raw cudaGraph_t): how many of
    the step's launches are ours. Returns (kernel_nodes, ours) or (None, None)."""
    try:
        import cuda.bindings.runtime as rt
        g = rt.cudaGraph_t(int(graph.raw_cuda_graph()))
        err, nodes, num = rt.cudaGraphGetNodes(g, 0)
        err, nodes, num = rt.cudaGraphGetNodes(g, num)
        kern = ours = 0
        for nd in nodes:
            err, ty = rt.cudaGraphNodeGetType(nd)
            if ty != rt.cudaGraphNodeType.cudaGraphNodeTypeKernel:
                continue
            kern += 1
            name = ""
            try:
                err, prm = rt.cudaGraphKernelNodeGetParams(nd)
                err, nm = rt.cudaFuncGetName(prm.func)
                name = nm.decode() if isinstance(nm, bytes) else str(nm)
            except Exception:  # noqa: BLE001
                pass
            if not name or any(k in name for k in ("onchip", "k_reduce", "k_ew", "k_finalize",
                                                     "k_fold", "k_coef", "p2p")):
                ours += 1
        return kern, ours
    except Exception:  # noqa: BLE001
        return None, None


# SURVEY 8(f) row 4 (producer fusion): the ResNet-50 1x1-conv -> BN layers of stages 1-2
# (H*W a multiple of 8), batch 32: (Cin, Cout, H, W, occurrences in the network)
PRODUCER_LAYERS = [(64, 64, 56, 56, 1), (256, 64, 56, 56, 2), (64, 256, 56, 56, 4),
                   (256, 128, 56, 56, 1), (512, 128, 28, 28, 3), (128, 512, 28, 28, 4)]


# channels_last producers: every conv->BN pair of torchvision ResNet-50 except the 7x7
# stem, (k, stride, Cin, Cout, H_in, W_in, occurrences); 52 of its 53 BN layers
PRODUCER_LAYERS_NHWC = [
    (1, 1, 64, 64, 56, 56, 1), (1, 1, 256, 64, 56, 56, 2), (3, 1, 64, 64, 56, 56, 3),
    (1, 1, 64, 256, 56, 56, 4),                                   # conv3 x3 + downsample
    (1, 1, 256, 128, 56, 56, 1), (3, 2, 128, 128, 56, 56, 1), (1, 2, 256, 512, 56, 56, 1),
    (1, 1, 512, 128, 28, 28, 3), (3, 1, 128, 128, 28, 28, 3), (1, 1, 128, 512, 28, 28, 4),
    (1, 1, 512, 256, 28, 28, 1), (3, 2, 256, 256, 28, 28, 1), (1, 2, 512, 1024, 28, 28, 1),
    (1, 1, 1024, 256, 14, 14, 5), (3, 1, 256, 256, 14, 14, 5), (1, 1, 256, 1024, 14, 14, 6),
    (1, 1, 1024, 512, 14, 14, 1), (3, 2, 512, 512, 14, 14, 1), (1, 2, 1024, 2048, 14, 14, 1),
    (1, 1, 2048, 512, 7, 7, 2), (3, 1, 512, 512, 7, 7, 2), (1, 1, 512, 2048, 7, 7, 3),
]


def producer_profile(cg, torch, dev, hbm_peak, batch=32, sets=3, iters=10):
    """Producer fusion on the tcgen05 1x1 conv: fused (conv epilogue emits the BN partial,
    then normalise) vs split (conv, then the BN forward re-reads z for its statistics),
    fp32 z, CUDA-graph timed with `sets` rotating buffer sets (no L2 reuse between
    launches). Totals are weighted by the layers' occurrences in ResNet-50."""
    from paper_1711_07240_b200 import producer as P

    def timed(fn):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                fn()
            g.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(iters):
                g.replay()
            e1.record(s)
            e1.synchronize()
        return e0.elapsed_time(e1) / iters / sets * 1e3  # us per layer

    tot = {"fused_us": 0.0, "split_us": 0.0, "conv_us": 0.0, "conv_bytes": 0}
    layers = []
    for cin, cout, h, w, cnt in PRODUCER_LAYERS:
        xs = [torch.randn(batch, cin, h, w, device=dev).to(torch.bfloat16) for _ in range(sets)]
        wt = (torch.randn(cout, cin, device=dev) / cin ** 0.5).to(torch.bfloat16)
        sts = [cg.BNLayerState.create(cout, device=dev) for _ in range(sets)]

        def conv():
            for x in xs:
                P.conv1x1(x, wt)

        def fused():
            for x, st in zip(xs, sts):
                P.conv1x1_bn_forward_local(x, wt, st)

        def split():
            for x, st in zip(xs, sts):
                cg.bn_forward_local(P.conv1x1(x, wt), st)

        w4 = wt[:, :, None, None]
        t_conv, t_f, t_s = timed(conv), timed(fused), timed(split)
        # the library baseline: cuDNN's conv (torch conv2d, bf16 out) + our BN forward, and
        # our fused conv with the same bf16 output
        t_cd = timed(lambda: [torch.nn.functional.conv2d(x, w4) for x in xs])
        t_cds = timed(lambda: [cg.bn_forward_local(torch.nn.functional.conv2d(x, w4), st)
                               for x, st in zip(xs, sts)])
        t_f16 = timed(lambda: [P.conv1x1_bn_forward_local(x, wt, st, out_dtype=torch.bfloat16)
                               for x, st in zip(xs, sts)])
        cb = batch * h * w * (2 * cin + 4 * cout) + 2 * cin * cout
        layers.append({"shape": [batch, cin, cout, h, w], "count": cnt, "conv_us": t_conv,
                       "conv_hbm_frac": cb / t_conv / 1e3 / hbm_peak,
                       "fused_fwd_us": t_f, "split_fwd_us": t_s, "cudnn_conv_us": t_cd,
                       "cudnn_split_fwd_us": t_cds, "fused_bf16_fwd_us": t_f16})
        tot["fused_us"] += cnt * t_f
        tot["split_us"] += cnt * t_s
        tot["conv_us"] += cnt * t_conv
        tot["conv_bytes"] += cnt * cb
        tot["cudnn_split_us"] = tot.get("cudnn_split_us", 0.0) + cnt * t_cds
        tot["fused_bf16_us"] = tot.get("fused_bf16_us", 0.0) + cnt * t_f16
        del xs, sts
    # channels_last (NHWC x and z): 1x1 and 3x3 over all stages
    cl = torch.channels_last
    ntot = {"fused_us": 0.0, "split_us": 0.0, "conv_us": 0.0}
    nlayers = []
    for k, sd, cin, cout, h, w, cnt in PRODUCER_LAYERS_NHWC:
        xs = [torch.randn(batch, cin, h, w, device=dev).to(torch.bfloat16).contiguous(
            memory_format=cl) for _ in range(sets)]
        # channels_last weights too, as model.to(memory_format=channels_last) leaves them
        wt = (torch.randn(cout, cin, k, k, device=dev) / (k * k * cin) ** 0.5).to(
            torch.bfloat16).contiguous(memory_format=cl)
        sts = [cg.BNLayerState.create(cout, device=dev) for _ in range(sets)]
        conv = P.conv3x3 if k == 3 else P.conv1x1
        fused_fn = P.conv3x3_bn_forward_local if k == 3 else P.conv1x1_bn_forward_local
        t_conv = timed(lambda: [conv(x, wt, stride=sd) for x in xs])
        t_f = timed(lambda: [fused_fn(x, wt, st, stride=sd) for x, st in zip(xs, sts)])
        t_s = timed(lambda: [cg.bn_forward_local(conv(x, wt, stride=sd), st)
                             for x, st in zip(xs, sts)])
        pad = k // 2
        t_cd = timed(lambda: [torch.nn.functional.conv2d(x, wt, stride=sd, padding=pad)
                              for x in xs])
        t_cds = timed(lambda: [cg.bn_forward_local(
            torch.nn.functional.conv2d(x, wt, stride=sd, padding=pad), st)
            for x, st in zip(xs, sts)])
        t_f16 = timed(lambda: [fused_fn(x, wt, st, stride=sd, out_dtype=torch.bfloat16)
                               for x, st in zip(xs, sts)])
        flops = 2.0 * batch * (h // sd) * (w // sd) * cout * cin * k * k
        nlayers.append({"k": k, "stride": sd, "shape": [batch, cin, cout, h, w], "count": cnt,
                        "conv_us": t_conv, "conv_tflops": flops / t_conv / 1e6,
                        "fused_fwd_us": t_f, "split_fwd_us": t_s, "cudnn_conv_us": t_cd,
                        "cudnn_conv_tflops": flops / t_cd / 1e6, "cudnn_split_fwd_us": t_cds,
                        "fused_bf16_fwd_us": t_f16})
        ntot["fused_us"] += cnt * t_f
        ntot["split_us"] += cnt * t_s
        ntot["conv_us"] += cnt * t_conv
        ntot["cudnn_split_us"] = ntot.get("cudnn_split_us", 0.0) + cnt * t_cds
        ntot["fused_bf16_us"] = ntot.get("fused_bf16_us", 0.0) + cnt * t_f16
        ntot["cudnn_conv_us"] = ntot.get("cudnn_conv_us", 0.0) + cnt * t_cd
        del xs, sts
    return {
        "what": "conv (tcgen05, bf16 x/w, fp32 z) + BN forward; fused = conv epilogue "
                "emits the BN partial (no statistics read of z), split = conv then the BN "
                "forward's statistics kernel re-reads z",
        "layers": "ResNet-50 stage 1-2 1x1-conv->BN layers (NCHW), batch 32, weighted by count",
        "fused_fwd_ms": tot["fused_us"] / 1e3, "split_fwd_ms": tot["split_us"] / 1e3,
        "speedup": tot["split_us"] / tot["fused_us"],
        "vs_cudnn": {"what": "bf16 z: our fused conv+BN forward vs cuDNN's conv (torch conv2d) "
                             "followed by our BN forward",
                     "fused_bf16_fwd_ms": tot["fused_bf16_us"] / 1e3,
                     "cudnn_split_fwd_ms": tot["cudnn_split_us"] / 1e3,
                     "speedup": tot["cudnn_split_us"] / tot["fused_bf16_us"]},
        "conv_gbs": tot["conv_bytes"] / tot["conv_us"] / 1e3,
        "conv_hbm_frac": tot["conv_bytes"] / tot["conv_us"] / 1e3 / hbm_peak,
        "per_layer": layers,
        "channels_last": {
            "layers": "every conv->BN pair of ResNet-50 but the 7x7 stem (52 of 53 BN layers; "
                      "1x1 and 3x3, stride 1 and 2; 3x3 / strided: implicit GEMM over TMA "
                      "im2col), NHWC, batch 32, weighted by count",
            "fused_fwd_ms": ntot["fused_us"] / 1e3, "split_fwd_ms": ntot["split_us"] / 1e3,
            "speedup": ntot["split_us"] / ntot["fused_us"],
            "conv_ms": ntot["conv_us"] / 1e3,
            "vs_cudnn": {"fused_bf16_fwd_ms": ntot["fused_bf16_us"] / 1e3,
                         "cudnn_split_fwd_ms": ntot["cudnn_split_us"] / 1e3,
                         "cudnn_conv_ms": ntot["cudnn_conv_us"] / 1e3,
                         "speedup": ntot["cudnn_split_us"] / ntot["fused_bf16_us"]},
            "per_layer": nlayers,
        },
    }


def select_transport(cg, torch, dist, dev, world, requested, barrier):
    """Statistics transport for N>1: NCCL all-gather, or the one-shot P2P exchange when it
    passes a self-test against NCCL (bitwise-equal rows, no timeout) and -- for "auto" --
    is faster. Every rank takes the same decision (collective MIN / MAX). Returns
    (handle, report)."""
    hn = cg.DistHandle(bn_group_size=world, transport="nccl")

    def time_exchange(h, c, reps=200):
        v = torch.zeros(2 * c + 1, dtype=torch.float64, device=dev)
        for _ in range(5):
            h.exchange(cg.SCOPE_BN_GROUP, "probe", v)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            h.exchange(cg.SCOPE_BN_GROUP, "probe", v)
        e1.record()
        torch.cuda.synchronize()
        tt = torch.tensor([e0.elapsed_time(e1) * 1e3 / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    rep = {"requested": requested}
    rep["nccl"] = {f"C{c}_us": time_exchange(hn, c) for c in (256, 2048)}
    rep["nccl"]["how"] = "all_gather_into_tensor of the fp64 partial (2C+1), eager"
    hp, ok = None, 0  # the self-test runs only if every rank set the P2P handle up
    if requested in ("auto", "p2p", "p2p_fused"):
        try:
            # auto and p2p_fused set the regions up for the fused variant too (G <= 8); a
            # p2p_fused handle also serves plain P2P exchanges
            fused_ok = requested in ("auto", "p2p_fused") and world <= 8
            hp = cg.DistHandle(bn_group_size=world,
                               transport="p2p_fused" if fused_ok else "p2p",
                               p2p_timeout_s=1.0)
            ok = 1
        except Exception as exc:  # noqa: BLE001
            rep["p2p_error"] = repr(exc)[:300]
        t = torch.tensor([ok], device=dev, dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)  # every rank set up, or nobody uses it
        ok = int(t.item())
    if ok:
        try:
            gen = torch.Generator(device=dev)
            gen.manual_seed(99 + dist.get_rank())
            good = True
            for c in (64, 2048, 64):
                v = torch.randn(2 * c + 1, dtype=torch.float64, device=dev, generator=gen)
                rp, _ = hp.exchange(cg.SCOPE_BN_GROUP, "selftest", v)
                rn, _ = hn.exchange(cg.SCOPE_BN_GROUP, "selftest", v)
                good = good and all(torch.equal(a, b) for a, b in zip(rp, rn))
            cg.check_status(dev)  # raises on an exchange timeout
            ok = int(good)
        except Exception as exc:  # noqa: BLE001 - reported; NCCL stays available
            rep["p2p_error"] = repr(exc)[:300]
            ok = 0
        t = torch.tensor([ok], device=dev, dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = int(t.item())
    if ok and hp.transport == "p2p_fused":
        # the fused path (push in the reduction, wait in the finalize) through the BN API:
        # bitwise equal to the NCCL path (every rank reaches the vote below)
        fgood = 0
        try:
            xs = torch.randn(4, 64, 14, 14, device=dev, generator=gen)
            st_f = cg.BNLayerState.create(64, device=dev)
            st_n = cg.BNLayerState.create(64, device=dev)
            y_f, c_f = cg.sync_bn_forward(hp, xs, st_f)
            y_n, c_n = cg.sync_bn_forward(hn, xs, st_n)
            dx_f = cg.sync_bn_backward(hp, xs, c_f, st_f)[0]
            dx_n = cg.sync_bn_backward(hn, xs, c_n, st_n)[0]
            cg.check_status(dev)
            fgood = int(torch.equal(y_f, y_n) and torch.equal(dx_f, dx_n))
        except Exception as exc:  # noqa: BLE001
            rep["p2p_fused_error"] = repr(exc)[:300]
        tf = torch.tensor([fgood], device=dev, dtype=torch.int32)
        dist.all_reduce(tf, op=dist.ReduceOp.MIN)
        fgood = int(tf.item())
        rep["p2p_fused_selftest"] = "passed" if fgood else "failed"
        if not fgood:
            hp.transport = "p2p"  # plain P2P exchanges; fused_exchange -> None
            if requested == "p2p_fused":
                ok = 0
    if requested in ("auto", "p2p", "p2p_fused"):
        rep["p2p_selftest"] = "passed" if ok else "failed"
        if ok:
            rep["p2p"] = {f"C{c}_us": time_exchange(hp, c) for c in (256, 2048)}
            rep["p2p"]["how"] = ("one single-CTA kernel per rank: NVLink pushes into CUDA-IPC "
                                 "regions, release/acquire epoch flags, eager")
    use_p2p = ok and (requested in ("p2p", "p2p_fused")
                      or rep["p2p"]["C256_us"] < rep["nccl"]["C256_us"])
    rep["step_transport"] = hp.transport if use_p2p else "nccl"
    if use_p2p and hp.transport == "p2p_fused":
        rep["p2p_fused_note"] = ("exchange fused into the kernels: the statistics reductions "
                                 "push into the regions, the finalize kernels wait "
                                 "(cgbn_*_p2p); the standalone P2P exchange latency is in "
                                 "'p2p'")
    if hp is not None and not use_p2p:
        hp.close()
    return (hp if use_p2p else hn), rep


def run_gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1711_07240_b200 as cg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torchrun (one rank per GPU)")
    # --same-device / --dist-backend gloo: every rank on GPU 0 with host-staged
    # exchanges, to exercise the N>1 orchestration on a single-GPU box (not a benchmark)
    dev_index = 0 if args.same_device else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    nccl = args.dist_backend == "nccl"
    if world > 1:
        if nccl:
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

        def _barrier():
            if nccl:
                dist.barrier(device_ids=[dev_index])
            else:
                dist.barrier()

        handle, transport_report = select_transport(cg, torch, dist, dev, world,
                                                    args.transport, _barrier)
    else:
        handle = cg.SoloHandle(dev)
        transport_report = None
    cg.set_strict(False)
    cg.set_fused(args.fused)

    shapes = WORKLOADS[args.workload][1]()
    elems = [numel(s) for s in shapes]
    # activation layout / dtype (default the reference's fp32 NCHW; channels_last and
    # bf16 are the SURVEY 8f row-2 widenings, reported as separate lines)
    act = {"f32": torch.float32, "bf16": torch.bfloat16}[args.act]
    esize = 4 if args.act == "f32" else 2
    mf = torch.channels_last if args.layout == "nhwc" else torch.contiguous_format
    lay = (_lib_consts().LAYOUT_NHWC if args.layout == "nhwc" else 0) | \
        (_lib_consts().ACT_BF16 if args.act == "bf16" else 0)
    bpe_step = BYTES_PER_ELEM * esize // 4
    step_bytes_rank = bpe_step * sum(elems)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    xs, dys, states = [], [], []
    for s in shapes:
        xs.append(torch.randn(s, device=dev, generator=gen).to(act).contiguous(memory_format=mf))
        dys.append(torch.randn(s, device=dev, generator=gen).to(act).contiguous(memory_format=mf))
        c = s[1]
        gamma = torch.rand(c, device=dev, generator=gen) + 0.5
        beta = torch.randn(c, device=dev, generator=gen)
        states.append(cg.BNLayerState(gamma=gamma, beta=beta))

    def step(xs_=None, dys_=None):
        xs_ = xs if xs_ is None else xs_
        dys_ = dys if dys_ is None else dys_
        caches = []
        for x, st in zip(xs_, states):
            _, cache = cg.sync_bn_forward(handle, x, st)
            caches.append(cache)
        for i in range(len(xs_) - 1, -1, -1):
            cg.sync_bn_backward(handle, dys_[i], caches[i], states[i])

    # L2 policy: a working set (x + dy of all layers) under 2x the L2 is replicated into
    # rotating input sets whose total exceeds 2x the L2, and the timed steps cycle through
    # them, so no step finds its inputs in L2 (and the timed region is back-to-back steps,
    # no per-step launch latency or flush inside it)
    ws_step = 2 * esize * sum(elems)
    n_sets = 1 if ws_step >= 2 * L2_BYTES else min(512, -(-2 * L2_BYTES // ws_step) + 1)
    sets = [(xs, dys)]
    for k in range(1, n_sets):
        sets.append(([x.clone() for x in xs], [d.clone() for d in dys]))

    def barrier():
        if world > 1:
            if nccl:
                dist.barrier(device_ids=[dev_index])
            else:
                dist.barrier()

    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(max(args.warmup, 3)):
            step()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()

    use_graph = not args.no_graph
    graph = None  # the one-step graph (its kernel nodes are counted)
    timed_graph = None  # rotating sets: one graph of all K timed steps
    graph_note = "cuda graph of the whole step" if use_graph else "eager"
    if use_graph:
        try:
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cap):  # the capture stream's workspace / status word
                step()                    # exist before capture (no fill kernels inside)
            torch.cuda.current_stream().wait_stream(cap)
            torch.cuda.synchronize()
            try:  # keep the cudaGraph_t after instantiation (kernel-node count)
                graph = torch.cuda.CUDAGraph(keep_graph=True)
            except TypeError:
                graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap):
                step()
            if n_sets > 1:
                # small working sets: the K timed steps cycle through the rotating input
                # sets inside ONE graph (one graph launch per timed region: a graph
                # launch per ~10 us step would make the host the bound)
                timed_graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(timed_graph, stream=cap):
                    for k in range(args.steps):
                        step(*sets[k % n_sets])
                graph_note = (f"cuda graph of the {args.steps} timed steps over {n_sets} "
                              "rotating input sets")
            for _ in range(2):
                (timed_graph or graph).replay()
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001 - e.g. a collective that cannot be captured
            print(f"[bench] graph capture failed ({exc!r}); timing eager steps", file=sys.stderr)
            graph = timed_graph = None
            graph_note = "eager (graph capture failed)"
            torch.cuda.synchronize()
            barrier()

    def run_once(k=0):
        if timed_graph is not None:
            if k == 0:
                timed_graph.replay()  # all K steps
        elif graph is not None:
            graph.replay()
        else:
            step(*sets[k % len(sets)])

    # ---- timed region
    if timed_graph is not None:
        # the warm replays left the graph's K input sets in L2 (K * ws_step can be far
        # under the L2 when K < n_sets): write a buffer of twice the L2 first, so the
        # timed graph starts cold; inside it no set is read twice
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
        flush.fill_(1.0)
        torch.cuda.synchronize()
        del flush
    sampler = ClockSampler(dev_index)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    l2_flush = n_sets > 1  # (rotating input sets; the name is kept for the config text)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for k in range(args.steps):
        run_once(k)
    t1.record()
    torch.cuda.synchronize()
    ms_total = t0.elapsed_time(t1)
    barrier()
    clocks = sampler.stop()
    if world > 1:
        tt = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / args.steps
    value = step_bytes_rank * world / (ms_step * 1e-3) / 1e9
    # our kernels per step: counted on the captured graph when there is one, else from
    # the plan (G == 1: one on-chip kernel or reduce + elementwise per direction; G > 1
    # adds the finalize kernel that folds the exchanged partials; NCCL not counted)
    from paper_1711_07240_b200 import _lib as _L
    on_f, on_b = _layer_paths(_L.load(), shapes, lay)
    if world == 1:
        planned = sum((1 if a else 2) + (1 if b else 2) for a, b in zip(on_f, on_b))
    else:
        planned = 6 * len(shapes)
    kern_nodes, ours = count_graph_kernels(graph) if graph is not None else (None, None)
    launches_per_step = ours if ours else planned

    # ---- per-kernel-family times: one CUDA graph per family replays that family's
    # launches of the step (same layer buffers, step order) through the C ABI
    kern, timing_mode = ({}, "skipped") if args.no_kprof else \
        kernel_profile(cg, shapes, xs, dys, states, handle, reps=20, lay=lay, esize=esize)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in peaks \
        else "fallback 6.65 TB/s (B200_PROFILING.md)"
    # the dominant family: by its share of the step in the committed ncu launch list
    # (profiles/r2_traffic.json: in-step, where L2 reuse between a reduction and its
    # elementwise pass counts), else by the direct family time
    dom, dom_by = None, None
    if kern:
        shares = {}
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "r2_traffic.json")))["families"]
            shares = {k: tr[k]["ncu_share"] for k in kern if k in tr}
        except Exception:  # noqa: BLE001
            pass
        if args.layout == "nchw" and args.act == "f32" and shares:
            dom, dom_by = max(shares, key=shares.get), "ncu in-step share (profiles/r2_traffic.json)"
        else:
            dom, dom_by = max(kern, key=lambda k: kern[k]["ms_per_step"]), "direct family time"
    roofline = None
    if dom:
        fam = kern[dom]
        ach = fam["alg_gbs"]
        traffic, tsrc = args.traffic, "--traffic"
        if traffic is None:
            traffic, tsrc = _traffic_for(dom, args.layout, args.act)
        t_launch = fam["ms_per_step"] * 1e-3 / fam["launches_per_step"]
        roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm_peak,
                    "unit": "GB/s", "frac": ach / hbm_peak, "traffic": traffic,
                    "traffic_unit": "ncu dram bytes (read + write) per launch",
                    "traffic_source": tsrc,
                    "dram_frac": (traffic / t_launch / 1e9 / hbm_peak) if traffic else None,
                    "alg_bytes_per_launch": fam["alg_bytes_per_launch"],
                    "alg_bytes_per_elem": fam["bytes_per_elem"],
                    "launches": fam["launches_per_step"], "us_per_launch": t_launch * 1e6,
                    "peak_source": peak_src, "timing": timing_mode, "dominant_by": dom_by,
                    "note": ("achieved = the family's algorithmic bytes per launch (on-chip "
                             "passes: their compulsory 8 / 12 B per element; split passes: "
                             "SURVEY 8d's 4 / 8 / 8 / 12) / its directly timed, L2-cold "
                             "launch time; dram_frac = ncu dram bytes per launch / that time")}

    # ---- statistics exchange latency (N>1): measured during transport selection
    exch = None
    if world > 1:
        exch = dict(transport_report)
        exch["per_step_exchanges"] = 2 * len(shapes)
        used = exch.get({"p2p_fused": "p2p"}.get(exch["step_transport"], exch["step_transport"]), {})
        if "C256_us" in used:
            exch["est_share_of_step"] = used["C256_us"] * 2 * len(shapes) * 1e-3 / ms_step

    # ---- e2e: public API with host (pinned) buffers, H2D/D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        def pinned(shape):  # pinned host buffer in the activation layout
            stride = torch.empty(shape, device="meta").contiguous(memory_format=mf).stride()
            return torch.empty_strided(shape, stride, dtype=act, pin_memory=True)

        hx = [pinned(s) for s in shapes]
        hdy = [pinned(s) for s in shapes]
        hy = [pinned(s) for s in shapes]
        hdx = [pinned(s) for s in shapes]
        for i in range(len(shapes)):
            hx[i].copy_(xs[i])
            hdy[i].copy_(dys[i])
        dx_in = [torch.empty(s, device=dev, dtype=act).contiguous(memory_format=mf)
                 for s in shapes]
        ddy_in = [torch.empty(s, device=dev, dtype=act).contiguous(memory_format=mf)
                  for s in shapes]

        # H2D on a copy-in stream, compute on the current stream, D2H on a copy-out stream
        # (the two PCIe directions run on separate copy engines), ordered by events: what
        # a caller staging host data through the public API would do.
        s_in = torch.cuda.Stream(device=dev)
        s_out = torch.cuda.Stream(device=dev)
        n_l = len(shapes)

        def e2e_step():
            comp = torch.cuda.current_stream(dev)
            ev_x = [torch.cuda.Event() for _ in range(n_l)]
            ev_dy = [torch.cuda.Event() for _ in range(n_l)]
            s_in.wait_stream(comp)  # the previous step is done with the input buffers
            with torch.cuda.stream(s_in):
                for i in range(n_l):
                    dx_in[i].copy_(hx[i], non_blocking=True)
                    ev_x[i].record(s_in)
                for i in range(n_l - 1, -1, -1):
                    ddy_in[i].copy_(hdy[i], non_blocking=True)
                    ev_dy[i].record(s_in)
            caches = []
            for i, st in enumerate(states):
                comp.wait_event(ev_x[i])
                y, cache = cg.sync_bn_forward(handle, dx_in[i], st)
                s_out.wait_stream(comp)
                with torch.cuda.stream(s_out):
                    hy[i].copy_(y, non_blocking=True)
                y.record_stream(s_out)
                caches.append(cache)
            for i in range(n_l - 1, -1, -1):
                comp.wait_event(ev_dy[i])
                dxo, dg, db = cg.sync_bn_backward(handle, ddy_in[i], caches[i], states[i])
                s_out.wait_stream(comp)
                with torch.cuda.stream(s_out):
                    hdx[i].copy_(dxo, non_blocking=True)
                dxo.record_stream(s_out)
            comp.wait_stream(s_out)  # the step ends when y and dx are in host memory

        # the drop-in default: strict device-status checks (a synchronous status read after
        # every public call, as the reference raises synchronously); --e2e-lenient times
        # set_strict(False) instead
        prev_strict = cg.set_strict(not args.e2e_lenient)
        for _ in range(3):  # warm-up (first touches of the pinned buffers)
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        k_e = max(10, args.e2e_steps)
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(k_e + 1)]
        marks[0].record()
        for k in range(k_e):
            e2e_step()
            marks[k + 1].record()
        torch.cuda.synchronize()
        barrier()
        cg.set_strict(prev_strict)
        ms_e_steps = [marks[k].elapsed_time(marks[k + 1]) for k in range(k_e)]
        ms_e = statistics.median(ms_e_steps)
        # the PCIe floor of the same step: the same H2D and D2H copies on the same two
        # streams with no compute between them (both directions concurrently)
        def copy_only_step(h2d=True, d2h=True):
            comp = torch.cuda.current_stream(dev)
            s_in.wait_stream(comp)
            s_out.wait_stream(comp)
            if h2d:
                with torch.cuda.stream(s_in):
                    for i in range(n_l):
                        dx_in[i].copy_(hx[i], non_blocking=True)
                    for i in range(n_l - 1, -1, -1):
                        ddy_in[i].copy_(hdy[i], non_blocking=True)
            if d2h:
                with torch.cuda.stream(s_out):
                    for i in range(n_l):
                        hy[i].copy_(xs[i], non_blocking=True)
                    for i in range(n_l - 1, -1, -1):
                        hdx[i].copy_(dys[i], non_blocking=True)
            comp.wait_stream(s_in)
            comp.wait_stream(s_out)

        def time_copies(**kw):
            copy_only_step(**kw)
            torch.cuda.synchronize()
            a0.record()
            for _ in range(k_e):
                copy_only_step(**kw)
            a1.record()
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / k_e

        # the PCIe floor of the step: each direction alone, and both at once (the e2e
        # step overlaps them, so max(h2d, d2h) is the bound it could reach)
        ms_h2d = time_copies(d2h=False)
        ms_d2h = time_copies(h2d=False)
        ms_both = time_copies()
        ms_copy = ms_both
        if world > 1:
            tt = torch.tensor([ms_e], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms_e = float(tt.item())
        e2e = {"value": step_bytes_rank * world / (ms_e * 1e-3) / 1e9, "unit": UNIT,
               "copy_only_ms_per_step": ms_copy,
               "copy_ms": {"h2d_alone": ms_h2d, "d2h_alone": ms_d2h, "both_at_once": ms_both},
               "pcie_gbs_per_direction": 2 * esize * sum(elems) / (ms_copy * 1e-3) / 1e9,
               "frac_of_copy_bound": ms_copy / ms_e,
               "frac_of_per_direction_bound": max(ms_h2d, ms_d2h) / ms_e,
               "copy_bound": "the step's H2D and D2H bytes copied at once on the same two "
                             "streams with no compute (both directions share the link: "
                             "measured slower than either alone, see copy_ms)",
               "h2d_bytes_per_step": 2 * esize * sum(elems),
               "d2h_bytes_per_step": 2 * esize * sum(elems),
               "ms_per_step": ms_e, "ms_mean": sum(ms_e_steps) / k_e, "steps": k_e,
               "statistic": "median of the timed steps (3 warm-up steps before)",
               "ms_each_step": ms_e_steps, "strict": not args.e2e_lenient,
               "path": "sync_bn_forward/sync_bn_backward per layer, eager (no graph), "
                       + ("strict status checks (the API default)" if not args.e2e_lenient
                          else "set_strict(False)")
                       + "; pinned host x/dy copied in on a copy-in stream, y/dx copied out on "
                       "a copy-out stream, event-ordered with the compute stream"}

    # ---- CPU baseline (rank 0, N=1 only): the reference on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = cpu_sample(shapes, 1, args.cpu_budget_s)
        cpu = {"value": res["gbs"], "unit": UNIT, "cores": 1, "kind": res["kind"],
               "sample": (f"{res['units']} {args.workload} BN layers at their own shapes "
                          f"(batch {shapes[0][0]}, from layer 0 on), f64, "
                          f"sync_bn_forward+backward via DeviceGroup(1); "
                          f"{res['seconds']:.1f} s"),
               **host_cpu_info()}

    parity = None
    if rank == 0 and not args.no_parity:
        try:
            parity = bench_parity(cg, torch, shapes, xs, dys, states, dev, esize)
        except Exception as exc:  # noqa: BLE001 - reported, never hides the line
            parity = {"ok": False, "error": f"{type(exc).__name__}: {exc}"}

    producer = None
    if rank == 0 and world == 1 and not args.no_producer:
        try:
            producer = producer_profile(cg, torch, dev, hbm_peak)
        except Exception as exc:  # report, never fail the bench line
            producer = {"error": f"{type(exc).__name__}: {exc}"}

    barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": f"{args.act} (fp64 statistics)", "data": "synthetic (torch.randn, seeded per rank)",
            "config": {"workload": args.workload, "describe": WORKLOADS[args.workload][0],
                       "layers": len(shapes),
                       "per_gpu_batch": shapes[0][0], "elements_per_gpu": sum(elems),
                       "alg_bytes_per_elem": bpe_step,
                       "parallelism": f"cgbn_group{world}", "bn_group_size": world,
                       "layout": args.layout.upper(), "relu": False,
                       "l2_policy": ((f"{n_sets} rotating input sets (x+dy = "
                                      f"{ws_step / 1e6:.1f} MB per step, {n_sets * ws_step / 1e6:.0f}"
                                      " MB in all > 2x the 126 MB L2): consecutive timed steps "
                                      "read different buffers, and a 2x-L2 write precedes the "
                                      "timed graph")
                                     if l2_flush else
                                     (f"inputs > L2: {len(shapes)} layers' x+dy = "
                                      f"{2 * esize * sum(elems) / 1e9:.2f} GB per step >> 126 MB L2; "
                                      "intra-layer re-reads of x may hit L2")),
                       "cuda_graph": graph is not None, "launch": graph_note,
                       "exchange_transport": (transport_report or {}).get(
                           "step_transport", "none (one rank)")},
            "per_gpu_gbs": value / world,
            "per_gpu_hbm_frac": value / world / hbm_peak,
            "kernels": kern,
            "t_fwd_ms": sum(v["ms_per_step"] for k, v in kern.items() if k.startswith("fwd"))
            if kern else None,
            "t_bwd_ms": sum(v["ms_per_step"] for k, v in kern.items() if k.startswith("bwd"))
            if kern else None,
            "layer_paths": {"fwd_onchip_layers": sum(on_f), "bwd_onchip_layers": sum(on_b),
                            "layers": len(shapes)},
            "graph_kernel_nodes": kern_nodes,
            "parity": parity,
            "roofline": roofline,
            "exchange": exch,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "producer_fusion": producer,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["cgbn", "reference"], default="cgbn")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help=argparse.SUPPRESS)  # gloo: orchestration test on one GPU
    ap.add_argument("--same-device", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--transport", choices=["auto", "nccl", "p2p", "p2p_fused"], default="auto",
                    help="BN-group statistics exchange at N>1: NCCL all-gather, the one-shot "
                         "P2P exchange, the P2P exchange fused into the reduction / finalize "
                         "kernels, or auto (P2P if it passes its self-test and is faster than "
                         "NCCL; fused when that also passes its BN-level self-test)")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="resnet50_bn_b32",
                    help="SURVEY 8(d) configuration (default: config 2, the driver's)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--layout", choices=["nchw", "nhwc"], default="nchw",
                    help="activation layout (nhwc = channels_last; SURVEY 8f row 2)")
    ap.add_argument("--act", choices=["f32", "bf16"], default="f32",
                    help="activation dtype (statistics stay fp64)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes/launch of the dominant kernel (recorded as-is)")
    ap.add_argument("--fused", action="store_true",
                    help="single-launch cooperative kernels for layers that fit on chip")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kprof", action="store_true", help="skip the per-kernel profile")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-lenient", action="store_true",
                    help="time e2e with set_strict(False) instead of the API default")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the post-timing oracle check of three of the timed layers")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-producer", action="store_true",
                    help="skip the producer-fusion (conv epilogue statistics) measurement")
    ap.add_argument("--ref-procs", type=int, default=None,
                    help="reference arm worker processes (default: one per allowed core)")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
