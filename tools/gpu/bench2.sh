#!/bin/bash
set -u
O=${1:-gpurun_out/bench2}
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 --no-producer > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --workload latency_2048x7x7 --no-producer > $O/bench_latency.json 2> $O/bench_latency.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
