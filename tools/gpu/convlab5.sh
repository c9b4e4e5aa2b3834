#!/bin/bash
set -u
O=${1:-gpurun_out/convlab5}
mkdir -p $O
timeout 900 python tools/conv_lab.py > $O/lab.jsonl 2> $O/lab.err
echo done >> $O/lab.err
