#!/bin/bash
set -u
O=${1:-gpurun_out/check5}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_conv_variants.py -q > $O/variants.log 2>&1; echo "rc=$?" >> $O/variants.log
timeout 300 python bench.py --workload latency_2048x7x7 --no-producer --no-cpu-baseline --no-e2e > $O/lat_default.json 2> $O/lat_default.err
timeout 300 python bench.py --workload latency_2048x7x7 --steps 20 --warmup 5 --no-producer --no-cpu-baseline --no-e2e > $O/lat_20.json 2> $O/lat_20.err
echo done > $O/done
