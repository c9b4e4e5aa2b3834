# bench the in-tree library against variant builds (CGBN_LIB) on three workloads
for w in resnet50_bn_b32 fpn_neck_800x1333 megdet_r50fpn_800x1333; do
  timeout 300 python bench.py --workload $w --steps 30 --no-e2e --no-cpu-baseline --no-kprof > gpurun_out/bl_base_$w.json 2>/dev/null
  for v in ewu1 ewu2; do
    CGBN_LIB=tools/bin/libcgbn_$v.so timeout 300 python bench.py --workload $w --steps 30 --no-e2e --no-cpu-baseline --no-kprof > gpurun_out/bl_${v}_$w.json 2>/dev/null
  done
done
