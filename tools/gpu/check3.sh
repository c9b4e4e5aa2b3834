#!/bin/bash
set -u
O=${1:-gpurun_out/check3}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --act bf16 --no-producer --no-cpu-baseline --no-e2e > $O/bench_bf16.json 2> $O/bench_bf16.err
timeout 600 python bench.py --steps 20 --warmup 5 --act bf16 --layout nhwc --no-producer --no-cpu-baseline --no-e2e > $O/bench_bf16_nhwc.json 2> $O/bench_bf16_nhwc.err
timeout 300 python tools/kbench.py --graph --iters 20 --dtype bf16 > $O/kb_bf16.jsonl 2> $O/kb_bf16.err
