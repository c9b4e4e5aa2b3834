#!/bin/bash
# channels_last row reductions: channel-slice width (CGBN_ROWS_CS4 float4 units) A/B on the
# fp32 and bf16 channels_last lines; "plan" = the planner's choice (32 up to C=256, else 64)
set -u
O=${1:-gpurun_out/cs4_ab}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
for v in plan 32 64 128; do
  L=""; [ $v != plan ] && L="CGBN_ROWS_CS4=$v"
  env $L timeout 300 python bench.py $Q --layout nhwc > $O/nhwc_f32_$v.json 2> $O/nhwc_f32_$v.err
  env $L timeout 300 python bench.py $Q --layout nhwc --act bf16 > $O/nhwc_bf16_$v.json 2> $O/nhwc_bf16_$v.err
done
echo done > $O/done
