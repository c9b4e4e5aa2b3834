#!/bin/bash
set -u
O=${1:-gpurun_out/trace2}
mkdir -p $O
timeout 300 python tools/onchip_trace.py --shape 32,128,28,28 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,64,56,56 --shape 32,512,7,7 > $O/trace.jsonl 2> $O/trace.err
timeout 300 python tools/kbench.py --graph --iters 20 > $O/kb_default.jsonl 2> $O/kb_default.err
timeout 600 python -m pytest tests/test_gpu_bench_shapes.py -q -x -k "shapes and 1-" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
