#!/bin/bash
# on-chip kernel: config sweep (graph-timed through the C ABI) + one ncu --set full capture
set -u
O=gpurun_out/onchip1
mkdir -p $O
for sh in 32,128,28,28 32,2048,7,7 32,1024,14,14 32,256,14,14; do
  for f in "" 1,2 1,4 2,4 2,2 4,2 8,1 16,1 4,1 2,1 1,1; do
    CGBN_ONCHIP_FORCE=$f CGBN_DEBUG_PLAN=1 timeout 120 python tools/kbench.py --graph --iters 20 --shape $sh \
      > $O/kb_${sh}_${f}.jsonl 2> $O/kb_${sh}_${f}.err
  done
done
K="python tools/kbench.py --shape 32,128,28,28 --iters 1"
$K > $O/kb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:k_onchip -s 0 -c 16 -o $O/onchip $K > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/onchip.ncu-rep > $O/summary.txt 2>&1
ncu -i $O/onchip.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null
ls -la $O | tail -3
