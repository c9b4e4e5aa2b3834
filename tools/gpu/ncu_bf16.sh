#!/bin/bash
# ncu --set full of the bf16 NCHW statistics and dx kernels on [32,256,56,56]
set -u
O=${1:-gpurun_out/ncu_bf16}
mkdir -p $O
timeout 300 python tools/kbench.py --dtype bf16 --shape 32,256,56,56 --iters 5 > $O/kb.jsonl 2> $O/kb.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_reduce|k_ew_dx" \
  --launch-skip 20 --launch-count 3 -o $O/bf16 -f \
  python tools/kbench.py --dtype bf16 --shape 32,256,56,56 --iters 5 > $O/ncu.log 2>&1; echo "rc=$?" >> $O/ncu.log
echo done > $O/done
