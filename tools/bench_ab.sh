# bench A/B of an env switch on the four workloads, 2 repetitions each
V=$1
for w in resnet50_bn_b32 fpn_neck_800x1333 megdet_r50fpn_800x1333; do
  for rep in 1 2; do
    timeout 300 python bench.py --workload $w --steps 30 --no-e2e --no-cpu-baseline --no-kprof > gpurun_out/bw_a_${w}_$rep.json 2>/dev/null
    env $V=1 timeout 300 python bench.py --workload $w --steps 30 --no-e2e --no-cpu-baseline --no-kprof > gpurun_out/bw_b_${w}_$rep.json 2>/dev/null
  done
done
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
