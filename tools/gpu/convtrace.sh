#!/bin/bash
set -u
O=${1:-gpurun_out/convtrace}
mkdir -p $O
for S in 1 2; do
CGBN_CONV_SPLITS=$S CGBN_CONV_TBN=128 timeout 120 python tools/conv_trace.py --layer 1,1,1024,256,14 > $O/t_1024_s$S.json 2>&1
CGBN_CONV_SPLITS=$S CGBN_CONV_TBN=128 timeout 120 python tools/conv_trace.py --layer 3,1,512,512,7 > $O/t_3x3_512_s$S.json 2>&1
done
echo done > $O/done
