#!/bin/bash
# Cout=64 layers: per-unit timelines (mainloop vs epilogue), planned and pinned tile widths,
# then one ncu --set full capture of the 3x3 64-channel conv on the current build.
set -u
O=${1:-gpurun_out/trace64}
mkdir -p $O
timeout 120 python tools/conv_trace.py --layer 3,1,64,64,56 > $O/t_3x3_64.json 2>&1
CGBN_CONV_TBN=128 timeout 120 python tools/conv_trace.py --layer 3,1,64,64,56 > $O/t_3x3_64_tbn128.json 2>&1
timeout 120 python tools/conv_trace.py --layer 1,1,256,64,56 > $O/t_256_64.json 2>&1
CGBN_CONV_TBN=256 timeout 120 python tools/conv_trace.py --layer 1,1,256,64,56 > $O/t_256_64_tbn256.json 2>&1
timeout 120 python tools/conv_trace.py --layer 1,1,64,256,56 > $O/t_64_256.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv \
  --launch-skip 6 --launch-count 1 -o $O/conv3x3_64 -f \
  python tools/conv_once.py 32,64,64,56,56 bf16 nhwc3 > $O/ncu.log 2>&1; echo "rc=$?" >> $O/ncu.log
echo done > $O/done
