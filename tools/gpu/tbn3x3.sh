#!/bin/bash
# 3x3 layers (and the Cout=64 set) with the tile width planned / pinned to 128 / 256.
set -u
O=${1:-gpurun_out/tbn3x3}
mkdir -p $O
timeout 300 python tools/conv_lab.py --layers 3x3 > $O/plan.jsonl 2>> $O/lab.err
CGBN_CONV_TBN=128 timeout 300 python tools/conv_lab.py --layers 3x3 > $O/t128.jsonl 2>> $O/lab.err
CGBN_CONV_TBN=256 timeout 300 python tools/conv_lab.py --layers 3x3 > $O/t256.jsonl 2>> $O/lab.err
CGBN_CONV_TBN=128 timeout 300 python tools/conv_lab.py --layers c64 > $O/c64_t128.jsonl 2>> $O/lab.err
CGBN_CONV_TBN=256 timeout 300 python tools/conv_lab.py --layers c64 > $O/c64_t256.jsonl 2>> $O/lab.err
echo done >> $O/lab.err
