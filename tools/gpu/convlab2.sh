#!/bin/bash
# producer conv: parity tests, then the lab with the planned tile width and with each
# width pinned
set -u
O=${1:-gpurun_out/convlab2}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 600 python tools/conv_lab.py > $O/lab_plan.jsonl 2> $O/lab.err
CGBN_CONV_TBN=128 timeout 600 python tools/conv_lab.py > $O/lab_128.jsonl 2>> $O/lab.err
CGBN_CONV_TBN=256 timeout 600 python tools/conv_lab.py > $O/lab_256.jsonl 2>> $O/lab.err
echo done >> $O/lab.err
