#!/bin/bash
# on-chip kernel: parity at the bench shapes (G=1 takes the on-chip path) + config sweep
set -u
O=${1:-gpurun_out/onchip2}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_bench_shapes.py -q -x -k "shapes and 1-" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x > $O/parity2.log 2>&1; echo rc=$? >> $O/parity2.log
CGBN_DEBUG_PLAN=1 timeout 300 python tools/kbench.py --graph --iters 20 > $O/kb_default.jsonl 2> $O/kb_default.err
for sh in 32,128,28,28 32,2048,7,7 32,1024,14,14 32,256,14,14 32,64,56,56 32,512,7,7; do
  for f in 1,1 1,2 1,4 1,8 2,1 2,2 2,4 4,1 4,2 8,1 16,1 32,1; do
    CGBN_ONCHIP_FORCE=$f CGBN_DEBUG_PLAN=1 timeout 120 python tools/kbench.py --graph --iters 20 --shape $sh \
      > $O/kb_${sh}_${f}.jsonl 2> $O/kb_${sh}_${f}.err
  done
done
