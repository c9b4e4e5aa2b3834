#!/bin/bash
set -u
O=${1:-gpurun_out/convlab9}
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for S in 2 3 4; do
CGBN_CONV_SPLITS=$S CGBN_CONV_TBN=128 timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_s$S.log 2>&1; echo "rc=$?" >> $O/tests_s$S.log
done
for S in 1 2 3 4; do
CGBN_CONV_SPLITS=$S CGBN_CONV_TBN=128 timeout 600 python tools/conv_lab.py --layers small > $O/lab_s$S.jsonl 2>> $O/lab.err
done
timeout 900 python tools/conv_lab.py > $O/lab.jsonl 2>> $O/lab.err
echo done >> $O/lab.err
