#!/bin/bash
# producer conv with CTA pairs: parity with pairs forced, then the lab (planned, and with
# the pair / tile width pinned)
set -u
O=${1:-gpurun_out/convlab3}
mkdir -p $O
CGBN_CONV_PAIR=1 timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_pair.log 2>&1; echo "rc=$?" >> $O/tests_pair.log
CGBN_CONV_PAIR=1 CGBN_CONV_TBN=256 timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_pair256.log 2>&1; echo "rc=$?" >> $O/tests_pair256.log
timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests_plan.log 2>&1; echo "rc=$?" >> $O/tests_plan.log
timeout 600 python tools/conv_lab.py > $O/lab_plan.jsonl 2> $O/lab.err
CGBN_CONV_PAIR=1 timeout 600 python tools/conv_lab.py > $O/lab_pair.jsonl 2>> $O/lab.err
CGBN_CONV_PAIR=1 CGBN_CONV_TBN=256 timeout 600 python tools/conv_lab.py > $O/lab_pair256.jsonl 2>> $O/lab.err
CGBN_CONV_PAIR=1 CGBN_CONV_TBN=128 timeout 600 python tools/conv_lab.py > $O/lab_pair128.jsonl 2>> $O/lab.err
echo done >> $O/lab.err
