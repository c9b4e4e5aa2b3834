#!/bin/bash
# channels_last 16-bit elementwise in fp32 when a thread's units share their channels:
# GPU suite, then the channels_last bf16 bench line with / without (CGBN_NHWC_F64=1), twice
set -u
O=${1:-gpurun_out/nhwc_f32}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for r in 1 2; do
timeout 600 python bench.py --layout nhwc --act bf16 --no-producer --no-cpu-baseline > $O/f32_$r.json 2> $O/f32_$r.err
CGBN_NHWC_F64=1 timeout 600 python bench.py --layout nhwc --act bf16 --no-producer --no-cpu-baseline > $O/f64_$r.json 2> $O/f64_$r.err
done
echo done > $O/done
