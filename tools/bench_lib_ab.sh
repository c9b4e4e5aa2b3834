# bench the in-tree library against variant builds (CGBN_LIB) on three workloads
for w in resnet50_bn_b32 fpn_neck_800x1333 megdet_r50fpn_800x1333; do
  timeout 300 python bench.py --workload $w --steps 30 --no-e2e --no-cpu-baseline --no-kprof > gpurun_out/bl_base_$w.json 2>/dev/null
  for v in vB vC vD; do
    CGBN_LIB=tools/bin/libcgbn_$v.so timeout 300 python bench.py --workload $w --steps 30 --no-e2e --no-cpu-baseline --no-kprof > gpurun_out/bl_${v}_$w.json 2>/dev/null
  done
done
S="--shape 32,64,56,56 --shape 32,256,56,56 --shape 32,128,28,28 --shape 32,1024,14,14 --shape 32,256,14,14 --shape 2,256,200,334"
timeout 300 python tools/kbench.py --graph $S > gpurun_out/blk_base.jsonl 2>&1
for v in vB vC vD; do CGBN_LIB=tools/bin/libcgbn_$v.so timeout 300 python tools/kbench.py --graph $S > gpurun_out/blk_$v.jsonl 2>&1; done
