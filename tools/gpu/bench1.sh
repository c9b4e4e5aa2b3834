#!/bin/bash
set -u
O=${1:-gpurun_out/bench1}
mkdir -p $O
timeout 300 python tools/onchip_trace.py --shape 32,128,28,28 --shape 32,256,14,14 --shape 32,2048,7,7 > $O/trace.jsonl 2> $O/trace.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-producer > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
CGBN_NO_ONCHIP=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity > $O/bench_split.json 2> $O/bench_split.err
