#!/bin/bash
# 64-row W boxes for Cout <= 64: producer parity, then the Cout=64 layers A/B.
set -u
O=${1:-gpurun_out/wrows}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_producer.py tests/test_gpu_conv_variants.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for r in 1 2; do
timeout 300 python tools/conv_lab.py --layers c64 > $O/lab_w64_$r.jsonl 2>> $O/lab.err
CGBN_CONV_WROWS=128 timeout 300 python tools/conv_lab.py --layers c64 > $O/lab_w128_$r.jsonl 2>> $O/lab.err
done
echo done >> $O/lab.err
