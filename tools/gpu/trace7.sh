#!/bin/bash
set -u
O=${1:-gpurun_out/trace7}
mkdir -p $O
timeout 300 python tools/onchip_trace.py --shape 32,128,28,28 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,64,56,56 > $O/trace.jsonl 2> $O/trace.err
timeout 300 python tools/kbench.py --graph --iters 20 > $O/kb_default.jsonl 2> $O/kb_default.err
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_invariants.py tests/test_gpu_p2p_fused.py tests/test_gpu_parity.py tests/test_gpu_half.py -q -x > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
