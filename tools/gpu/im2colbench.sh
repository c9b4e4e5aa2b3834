#!/bin/bash
set -u
O=${1:-gpurun_out/im2colbench}
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o $O/im2colbench tools/lab/im2colbench.cu > $O/build.log 2>&1
timeout 120 $O/im2colbench > $O/im2colbench.jsonl 2>&1; echo "rc=$?" >> $O/build.log
rm -f $O/im2colbench
