#!/bin/bash
# 16-bit on-chip passes (fp32 grouped reduction + fp32 write): forced-on-chip parity, then
# the bf16 ResNet-50 line at footprint caps 0 / 0.1 / 0.2 / 0.4
set -u
O=${1:-gpurun_out/onchip16}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_onchip.py tests/test_gpu_half.py -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline"
for f in 0 0.1 0.2 0.4; do
  CGBN_ONCHIP_MAX_FRAC=$f timeout 300 python bench.py $Q --act bf16 > $O/bf16_$f.json 2> $O/bf16_$f.err
done
echo done > $O/done
