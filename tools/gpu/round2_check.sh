#!/bin/bash
# GPU tests + bench lines of every workload (evidence for profiles/)
set -u
O=${1:-gpurun_out/r2check}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
for w in fpn_neck_800x1333 megdet_r50fpn_800x1333 latency_2048x7x7; do
  timeout 600 python bench.py --steps 20 --warmup 5 --workload $w --no-producer > $O/bench_$w.json 2> $O/bench_$w.err
done
for l in "--layout nhwc" "--act bf16" "--layout nhwc --act bf16"; do
  n=$(echo $l | tr -d ' -')
  timeout 600 python bench.py --steps 20 --warmup 5 $l --no-producer --no-cpu-baseline > $O/bench_$n.json 2> $O/bench_$n.err
done
