#!/bin/bash
set -u
O=${1:-gpurun_out/producer}
mkdir -p $O
timeout 1500 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-parity > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
