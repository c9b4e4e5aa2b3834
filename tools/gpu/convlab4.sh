#!/bin/bash
set -u
O=${1:-gpurun_out/convlab4}
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_plan.log 2>&1; echo "rc=$?" >> $O/tests_plan.log
CGBN_CONV_PAIR=1 timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_pair.log 2>&1; echo "rc=$?" >> $O/tests_pair.log
CGBN_CONV_PAIR=0 timeout 600 python tools/conv_lab.py > $O/lab_nopair.jsonl 2> $O/lab.err
CGBN_CONV_PAIR=1 timeout 600 python tools/conv_lab.py > $O/lab_pair.jsonl 2>> $O/lab.err
CGBN_CONV_PAIR=0 CGBN_CONV_TBN=128 timeout 600 python tools/conv_lab.py > $O/lab_128.jsonl 2>> $O/lab.err
CGBN_CONV_PAIR=0 CGBN_CONV_TBN=256 timeout 600 python tools/conv_lab.py > $O/lab_256.jsonl 2>> $O/lab.err
echo done >> $O/lab.err
