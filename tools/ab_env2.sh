# A/B of an env switch on big and mid shapes + the two detector workloads
V=$1
S="--shape 2,256,200,334 --shape 2,64,400,667 --shape 32,256,56,56 --shape 2,256,50,84 --shape 32,256,14,14"
timeout 300 python tools/kbench.py --graph $S > gpurun_out/kb_a.jsonl 2>&1
env $V=1 timeout 300 python tools/kbench.py --graph $S > gpurun_out/kb_b.jsonl 2>&1
for w in resnet50_bn_b32 megdet_r50fpn_800x1333; do
  timeout 300 python bench.py --workload $w --steps 30 --no-e2e --no-cpu-baseline --no-kprof > gpurun_out/bw_a_$w.json 2>/dev/null
  env $V=1 timeout 300 python bench.py --workload $w --steps 30 --no-e2e --no-cpu-baseline --no-kprof > gpurun_out/bw_b_$w.json 2>/dev/null
done
