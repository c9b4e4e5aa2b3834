#!/bin/bash
set -u
O=${1:-gpurun_out/red_ab3}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
for v in default red41; do
  L=""; [ $v != default ] && L="CGBN_LIB=paper_1711_07240_b200/libcgbn_$v.so"
  env $L timeout 300 python bench.py $Q > $O/f32_$v.json 2> $O/f32_$v.err
  env $L timeout 300 python bench.py $Q --act bf16 > $O/bf16_$v.json 2> $O/bf16_$v.err
done
echo done > $O/done
