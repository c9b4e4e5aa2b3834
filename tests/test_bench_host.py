"""bench.py host-side definitions (CPU): the SURVEY 8(d) workloads, the ResNet-50 BN
layer list, the reference-arm process sizing and the oracle fallback step."""

import bench


def test_resnet50_has_53_bn_layers_at_224():
    s = bench.resnet50_bn_shapes(32)
    assert len(s) == 53
    assert s[0] == (32, 64, 112, 112)
    assert s[-1] == (32, 2048, 7, 7)
    assert sum(bench.numel(x) for x in s) == 355_647_488


def test_detector_workloads_use_ceil_strides():
    fpn = bench.fpn_neck_shapes(2)
    assert fpn == [(2, 256, 200, 334), (2, 256, 100, 167), (2, 256, 50, 84),
                   (2, 256, 25, 42), (2, 256, 13, 21)]
    meg = bench.WORKLOADS["megdet_r50fpn_800x1333"][1]()
    assert len(meg) == 58 and meg[0] == (2, 64, 400, 667)
    assert bench.WORKLOADS["latency_2048x7x7"][1]() == [(1, 2048, 7, 7)]


def test_reference_procs_capped_by_cores():
    n = bench.reference_procs(bench.resnet50_bn_shapes(32), 1)
    assert 1 <= n <= (len(__import__("os").sched_getaffinity(0)))
    assert bench.reference_procs(bench.resnet50_bn_shapes(32), 1, requested=1) == 1


def test_port_step_counts_algorithmic_bytes():
    dt, nb = bench.port_step((2, 8, 4, 4), 2, 0)
    assert nb == 32 * 2 * 8 * 16 * 2 and dt > 0


def test_host_cpu_info_keys():
    info = bench.host_cpu_info()
    assert {"cpu_model", "host_cpus", "affinity_cpus"} <= set(info)


def test_reference_arm_json_line_contract():
    """`bench.py --impl reference` prints one JSON line with the reference-arm keys
    (CPU only: the arm times the reference's own CPU path, or the oracle port when
    baseline/_ref is absent)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run(
        [sys.executable, "bench.py", "--impl", "reference", "--workload", "latency_2048x7x7",
         "--steps", "2", "--warmup", "3", "--ref-procs", "1"],
        cwd=root, capture_output=True, text=True, timeout=300, check=True)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT and d["value"] > 0
    assert d["higher_is_better"] is True and d["n_gpus"] == 1
    # like-for-like with the GPU arm: the config's own workload and per-GPU batch
    assert d["config"]["workload"] == "latency_2048x7x7" and d["config"]["per_gpu_batch"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] == 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
