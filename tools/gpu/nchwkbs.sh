#!/bin/bash
set -u
O=${1:-gpurun_out/nchwkbs}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_producer.py tests/test_gpu_conv_variants.py -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-parity > $O/bench.json 2> $O/bench.err
echo done > $O/done
