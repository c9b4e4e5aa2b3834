#!/bin/bash
set -u
O=${1:-gpurun_out/convlab11}
mkdir -p $O
CGBN_CONV_SPLITS=2 CGBN_CONV_TBN=128 timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_s2.log 2>&1; echo "rc=$?" >> $O/tests_s2.log
for S in 1 2 4; do
CGBN_CONV_SPLITS=$S CGBN_CONV_TBN=128 timeout 600 python tools/conv_lab.py --layers small > $O/lab_s$S.jsonl 2>> $O/lab.err
done
echo done >> $O/lab.err
