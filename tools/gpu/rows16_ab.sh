#!/bin/bash
set -u
O=${1:-gpurun_out/rows16_ab}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
for v in default r16a r16b; do
  L=""; [ $v != default ] && L="CGBN_LIB=paper_1711_07240_b200/libcgbn_$v.so"
  env $L timeout 300 python bench.py $Q --layout nhwc --act bf16 > $O/nhwc_bf16_$v.json 2> $O/nhwc_bf16_$v.err
done
echo done > $O/done
