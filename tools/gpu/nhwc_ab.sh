#!/bin/bash
# A/B on the channels_last bench lines: current build vs the NHWC elementwise U=2 variant
set -u
O=${1:-gpurun_out/nhwc_ab}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
for v in default ewu2; do
  L=""; [ $v = ewu2 ] && L="CGBN_LIB=paper_1711_07240_b200/libcgbn_ewu2.so"
  env $L timeout 300 python bench.py $Q --layout nhwc > $O/nhwc_f32_$v.json 2> $O/nhwc_f32_$v.err
  env $L timeout 300 python bench.py $Q --layout nhwc --act bf16 > $O/nhwc_bf16_$v.json 2> $O/nhwc_bf16_$v.err
done
timeout 300 python tools/kbench.py --graph --nhwc --dtype bf16 --shape 32,256,56,56 --shape 32,1024,14,14 --shape 32,64,112,112 > $O/kb_nhwc_bf16.jsonl 2> $O/kb.err
timeout 600 python -m pytest tests -m gpu -q -x -k "nhwc or rows or channels_last or layout" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
echo done > $O/done
