#!/bin/bash
# conv lab: per-layer timing vs cuDNN, then one ncu --set full capture of the plain 3x3
# conv on [32,64,64,56,56] NHWC (bf16 out).
set -u
O=${1:-gpurun_out/convlab}
mkdir -p $O
timeout 900 python tools/conv_lab.py > $O/lab.jsonl 2> $O/lab.err; echo "rc=$?" >> $O/lab.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv1x1 \
  --launch-skip 6 --launch-count 1 -o $O/conv3x3_64 -f \
  python tools/conv_once.py 32,64,64,56,56 bf16 nhwc3 > $O/ncu.log 2>&1; echo "rc=$?" >> $O/ncu.log
