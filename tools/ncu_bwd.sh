# ncu --set full of the backward kernels (bwd cluster-team reduce, dx elementwise) at
# [32,256,56,56]; summarised on the box (reports can exceed gpurun's copy-back limit)
OUT=${1:-gpurun_out/prof_bwd}
mkdir -p $OUT
K="python tools/kbench.py --shape 32,256,56,56 --iters 3"
$K > $OUT/kb_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"k_reduce_ct<.*BwdOp" -c 1 -o $OUT/bwd_reduce $K > $OUT/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"k_ew_dx" -c 1 -o $OUT/dx $K > $OUT/ncu2.log 2>&1
for r in $OUT/bwd_reduce.ncu-rep $OUT/dx.ncu-rep; do
  [ -f "$r" ] && python tools/ncu_summary.py "$r" >> $OUT/summary.txt 2>&1
done
rm -f $OUT/*.ncu-rep
