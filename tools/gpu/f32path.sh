#!/bin/bash
set -u
O=${1:-gpurun_out/f32path}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $Q --act bf16 > $O/bf16.json 2> $O/bf16.err
timeout 300 python bench.py $Q --act bf16 --layout nhwc > $O/nhwc_bf16.json 2> $O/nhwc_bf16.err
timeout 300 python tools/kbench.py --graph --dtype bf16 --shape 32,256,56,56 --shape 32,1024,14,14 > $O/kb_bf16.jsonl 2> $O/kb.err
timeout 300 python tools/kbench.py --graph --dtype bf16 --nhwc --shape 32,256,56,56 --shape 32,1024,14,14 > $O/kb_nhwc_bf16.jsonl 2>> $O/kb.err
echo done > $O/done
