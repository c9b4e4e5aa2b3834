#!/bin/bash
set -u
O=${1:-gpurun_out/trace6}
mkdir -p $O
timeout 300 python tools/onchip_trace.py --shape 32,128,28,28 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,64,56,56 > $O/trace.jsonl 2> $O/trace.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_dist_procs.py tests/test_gpu_fd.py tests/test_gpu_reference_mode.py tests/test_gpu_producer.py tests/test_gpu_p2p.py tests/test_gpu_nccl_graph.py -q -x > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
