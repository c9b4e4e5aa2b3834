#!/bin/bash
set -u
O=${1:-gpurun_out/convlab8}
mkdir -p $O
CGBN_CONV_SPLITS=2 timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_s2.log 2>&1; echo "rc=$?" >> $O/tests_s2.log
CGBN_CONV_SPLITS=3 CGBN_CONV_TBN=128 timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_s3.log 2>&1; echo "rc=$?" >> $O/tests_s3.log
timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python tools/conv_lab.py > $O/lab.jsonl 2> $O/lab.err
CGBN_CONV_SPLITS=1 timeout 900 python tools/conv_lab.py --layers small > $O/lab_s1.jsonl 2>> $O/lab.err
CGBN_CONV_SPLITS=2 CGBN_CONV_TBN=128 timeout 900 python tools/conv_lab.py --layers small > $O/lab_s2.jsonl 2>> $O/lab.err
CGBN_CONV_SPLITS=3 CGBN_CONV_TBN=128 timeout 900 python tools/conv_lab.py --layers small > $O/lab_s3.jsonl 2>> $O/lab.err
echo done >> $O/lab.err
