#!/bin/bash
# one ncu --set full capture (with source) of the plain NHWC conv on a given layer
set -u
O=${O:-gpurun_out/convprof}
mkdir -p $O
SHAPE=${SHAPE:-32,64,256,56,56}
MODE=${MODE:-nhwc1}
timeout 300 python tools/conv_once.py $SHAPE bf16 $MODE > $O/plain.log 2>&1; echo "rc=$?" >> $O/plain.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv1x1 \
  --launch-skip 6 --launch-count 1 -o $O/${TAG:-conv} -f \
  python tools/conv_once.py $SHAPE bf16 $MODE > $O/ncu.log 2>&1; echo "rc=$?" >> $O/ncu.log
