#!/bin/bash
set -u
O=${1:-gpurun_out/rows_ab}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
for v in default rows42; do
  L=""; [ $v = rows42 ] && L="CGBN_LIB=paper_1711_07240_b200/libcgbn_rows42.so"
  env $L timeout 300 python bench.py $Q --layout nhwc > $O/nhwc_$v.json 2> $O/nhwc_$v.err
  env $L timeout 300 python tools/kbench.py --graph --nhwc --shape 32,256,56,56 --shape 32,1024,14,14 --shape 32,128,28,28 > $O/kb_$v.jsonl 2> $O/kb_$v.err
done
echo done > $O/done
