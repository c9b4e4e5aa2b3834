#!/bin/bash
set -u
O=${1:-gpurun_out/minb}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
for v in default minb3; do
  L=""; [ $v = minb3 ] && L="CGBN_LIB=paper_1711_07240_b200/libcgbn_minb3.so"
  env $L timeout 300 python bench.py $Q > $O/resnet_$v.json 2> $O/resnet_$v.err
  env $L timeout 300 python bench.py $Q --act bf16 > $O/resnet_bf16_$v.json 2> $O/resnet_bf16_$v.err
  env $L timeout 300 python tools/kbench.py --graph --iters 20 > $O/kb_$v.jsonl 2> $O/kb_$v.err
done
