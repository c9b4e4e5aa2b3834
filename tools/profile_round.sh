#!/bin/bash
# One gpurun call's worth of evidence for profiles/ (run from the repo root on a B200):
# GPU tests, graph-mode per-kernel microbenchmarks, the full bench line, the ncu launch
# list of one bench step, and ncu --set full captures of the dominant kernels.
set -u
OUT=${1:-gpurun_out/prof_round}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python tools/kbench.py --graph > $OUT/kbench_graph.jsonl 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
# launch list of one eager step (cold caches not forced: --cache-control none keeps the
# step's own L2 state)
CMD="python bench.py --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-kprof"
$CMD > $OUT/step_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --cache-control none --clock-control none --csv --log-file $OUT/launches.csv $CMD \
      > $OUT/ncu_launches.log 2>&1
# full sets of the dominant kernels on the largest ResNet-50 shape
K="python tools/kbench.py --shape 32,256,56,56 --iters 3"
$K > $OUT/kb_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_ew_dx|k_reduce|k_ew_affine" \
      -s 0 -c 12 -o $OUT/full $K > $OUT/ncu_full.log 2>&1
K2="python tools/kbench.py --shape 32,128,28,28 --iters 3"
$K2 > $OUT/kb2_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_reduce" \
      -s 0 -c 4 -o $OUT/full_mid $K2 > $OUT/ncu_full_mid.log 2>&1
# summarise the full captures on the box (the .ncu-rep files can exceed gpurun's 64 MiB
# copy-back limit); keep only the mid-shape report
for r in $OUT/full.ncu-rep $OUT/full_mid.ncu-rep; do
  [ -f "$r" ] && python tools/ncu_summary.py "$r" >> $OUT/ncu_full_summary.txt 2>&1
done
rm -f $OUT/full.ncu-rep
du -sh $OUT
echo done
