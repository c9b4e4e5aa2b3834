#!/bin/bash
set -u
O=${1:-gpurun_out/trace3}
mkdir -p $O
timeout 300 python tools/onchip_trace.py --shape 32,128,28,28 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,64,56,56 --shape 32,512,7,7 --shape 1,2048,7,7 > $O/trace.jsonl 2> $O/trace.err
timeout 300 python tools/kbench.py --graph --iters 20 > $O/kb_default.jsonl 2> $O/kb_default.err
K="python tools/kbench.py --shape 32,256,14,14 --iters 1"
$K > $O/kb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:k_onchip -s 2 -c 2 -o $O/onchip $K > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/onchip.ncu-rep > $O/summary.txt 2>&1
ncu -i $O/onchip.ncu-rep --page source --csv --print-source sass > $O/source.csv 2>/dev/null
rm -f $O/onchip.ncu-rep
