#!/bin/bash
# A/B of the fused single-rank kernels: launch modes and the graph step (under gpurun).
S="--shape 32,128,28,28 --shape 32,256,14,14"
python tools/kbench.py $S > gpurun_out/ab_coop.jsonl 2>&1
CGBN_NO_COOP=1 python tools/kbench.py $S > gpurun_out/ab_nocoop.jsonl 2>&1
python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_bench_fused.json 2>&1
CGBN_NO_COOP=1 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_bench_nocoop.json 2>&1
CGBN_NO_FUSED=1 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_bench_split.json 2>&1
python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ab_bench_fused_eager.json 2>&1
python tools/kbench.py --shape 32,256,14,14 --iters 5 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/ab_fused_ncu.csv python tools/kbench.py --shape 32,256,14,14 --iters 5 > /dev/null 2>&1
echo done
