#!/bin/bash
# A/B profile of the register vs TMA kernel families on one shape (run under gpurun).
SHAPE=${1:-32,256,56,56}
python tools/kbench.py --shape $SHAPE --iters 5 > gpurun_out/ab_plain.log 2>&1 || exit 1
CGBN_PATH=reg python tools/kbench.py --shape $SHAPE --iters 5 > gpurun_out/ab_plain_reg.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 8 -o gpurun_out/prof_tma python tools/kbench.py --shape $SHAPE --iters 5 > gpurun_out/ab_ncu_tma.log 2>&1
CGBN_PATH=reg ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 8 -o gpurun_out/prof_reg python tools/kbench.py --shape $SHAPE --iters 5 > gpurun_out/ab_ncu_reg.log 2>&1
