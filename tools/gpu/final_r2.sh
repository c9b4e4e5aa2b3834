#!/bin/bash
# round-2 evidence: GPU tests, smoke, every bench line, reference arm
set -u
O=${1:-gpurun_out/final_r2}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
for w in fpn_neck_800x1333 megdet_r50fpn_800x1333 latency_2048x7x7; do
  timeout 600 python bench.py --workload $w --no-producer > $O/bench_$w.json 2> $O/bench_$w.err
done
for l in "--layout nhwc" "--act bf16" "--layout nhwc --act bf16"; do
  n=$(echo $l | tr -d ' -')
  timeout 600 python bench.py $l --no-producer --no-cpu-baseline > $O/bench_$n.json 2> $O/bench_$n.err
done
echo done > $O/done
