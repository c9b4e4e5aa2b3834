#!/bin/bash
set -u
O=${1:-gpurun_out/convlab12}
mkdir -p $O
bash tools/gpu/convtrace.sh $O
for S in 2 3; do
CGBN_CONV_SPLITS=$S CGBN_CONV_TBN=128 timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_s$S.log 2>&1; echo "rc=$?" >> $O/tests_s$S.log
done
timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python tools/conv_lab.py > $O/lab.jsonl 2> $O/lab.err
CGBN_CONV_SPLITS=1 timeout 900 python tools/conv_lab.py --layers small > $O/lab_small_s1.jsonl 2>> $O/lab.err
echo done >> $O/lab.err
