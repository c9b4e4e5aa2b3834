#!/bin/bash
set -u
O=${1:-gpurun_out/check2}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_onchip.py tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_invariants.py tests/test_gpu_bench_shapes.py -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --act bf16 --no-producer --no-cpu-baseline --no-e2e > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-producer --no-cpu-baseline > $O/bench.json 2> $O/bench.err
