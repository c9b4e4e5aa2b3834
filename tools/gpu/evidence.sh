#!/bin/bash
# ncu evidence for profiles/: the step's launch list (per-family DRAM traffic) and full
# captures of the kernels VERDICT r1 asked for (bwd reduce, dx, channels_last rows + fold,
# bf16 statistics) plus the on-chip kernels. Summaries are made on the box (the .ncu-rep
# files would exceed gpurun's copy-back limit).
set -u
O=${1:-gpurun_out/evidence}
mkdir -p $O
S="python bench.py --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-kprof --no-parity --no-producer"
$S > $O/step_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --cache-control none --clock-control none --csv --log-file $O/launches.csv $S \
      > $O/ncu_launches.log 2>&1
python tools/step_breakdown.py $O/launches.csv --traffic $O/r2_traffic.json --passes 4 > $O/step_breakdown.txt 2>&1
full() {  # name, kernel regex, count, command...
  local n=$1 k=$2 c=$3; shift 3
  "$@" > $O/${n}_plain.log 2>&1 && \
    ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k regex:"$k" -s 0 -c $c -o $O/$n "$@" > $O/${n}_ncu.log 2>&1
  python tools/ncu_summary.py $O/$n.ncu-rep >> $O/ncu_full_summary.txt 2>&1
  rm -f $O/$n.ncu-rep
}
full bwd "k_reduce_ct<.*BwdOp|k_ew_dx" 2 python tools/kbench.py --shape 32,256,56,56 --iters 1
full nhwc "k_reduce_rows|k_fold_rows" 4 python tools/kbench.py --shape 32,256,56,56 --iters 1 --nhwc
full bf16 "k_reduce_ct<.*StatsOp<__nv_bfloat16|k_ew_affine<__nv_bfloat16" 2 python tools/kbench.py --shape 32,256,56,56 --iters 1 --dtype bf16
full onchip "k_onchip" 2 python tools/kbench.py --shape 32,256,14,14 --iters 1
du -sh $O
