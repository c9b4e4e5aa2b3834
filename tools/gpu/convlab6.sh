#!/bin/bash
set -u
O=${1:-gpurun_out/convlab6}
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_producer.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 900 python tools/conv_lab.py > $O/lab.jsonl 2> $O/lab.err
echo done >> $O/lab.err
