#!/bin/bash
set -u
O=${1:-gpurun_out/lat5}
mkdir -p $O
timeout 300 python tools/onchip_trace.py --shape 1,2048,7,7 > $O/trace.jsonl 2> $O/trace.err
timeout 300 python tools/kbench.py --graph --shape 1,2048,7,7 > $O/kb.jsonl 2> $O/kb.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --workload latency_2048x7x7 --steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity --no-kprof > $O/ncu.log 2>&1
echo done > $O/done
