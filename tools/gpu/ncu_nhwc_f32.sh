#!/bin/bash
# channels_last bf16 normalise / dx, fp32 records vs fp64 coefficients: kbench + ncu --set full
set -u
O=${1:-gpurun_out/ncu_nhwc_f32}
mkdir -p $O
timeout 300 python tools/kbench.py --nhwc --dtype bf16 --shape 32,256,56,56 --iters 20 > $O/kb_f32.jsonl 2> $O/kb.err
CGBN_NHWC_F64=1 timeout 300 python tools/kbench.py --nhwc --dtype bf16 --shape 32,256,56,56 --iters 20 > $O/kb_f64.jsonl 2>> $O/kb.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ew_" \
  --launch-skip 10 --launch-count 4 -o $O/f32 -f \
  python tools/kbench.py --nhwc --dtype bf16 --shape 32,256,56,56 --iters 5 > $O/ncu_f32.log 2>&1; echo "rc=$?" >> $O/ncu_f32.log
CGBN_NHWC_F64=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ew_" \
  --launch-skip 10 --launch-count 4 -o $O/f64 -f \
  python tools/kbench.py --nhwc --dtype bf16 --shape 32,256,56,56 --iters 5 > $O/ncu_f64.log 2>&1; echo "rc=$?" >> $O/ncu_f64.log
echo done > $O/done
