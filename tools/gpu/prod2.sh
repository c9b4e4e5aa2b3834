#!/bin/bash
# two TMA-issuing threads per conv CTA: producer parity (every pinned variant), then the
# conv lab with 2 / 1 producers
set -u
O=${1:-gpurun_out/prod2}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_producer.py tests/test_gpu_conv_variants.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 600 python tools/conv_lab.py > $O/lab_p2.jsonl 2>> $O/lab.err
CGBN_CONV_PRODUCERS=1 timeout 600 python tools/conv_lab.py > $O/lab_p1.jsonl 2>> $O/lab.err
echo done >> $O/lab.err
