#!/bin/bash
# A/B on the bf16 NCHW bench line: elementwise units per thread 2 (default) vs 4
set -u
O=${1:-gpurun_out/bf16_ab}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
for v in default ewu4; do
  L=""; [ $v = ewu4 ] && L="CGBN_LIB=paper_1711_07240_b200/libcgbn_ewu4.so"
  env $L timeout 300 python bench.py $Q --act bf16 > $O/bf16_$v.json 2> $O/bf16_$v.err
  env $L timeout 300 python bench.py $Q > $O/f32_$v.json 2> $O/f32_$v.err
done
timeout 300 python bench.py $Q --workload latency_2048x7x7 > $O/lat.json 2> $O/lat.err
echo done > $O/done
