#!/bin/bash
# in-step A/B of the on-chip passes: the footprint cap (fraction of the GPU's shared memory)
set -u
O=${1:-gpurun_out/onchip_frac}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity --no-kprof"
for f in 0 0.03 0.06 0.1 0.2 0.4 0.8; do
  CGBN_ONCHIP_MAX_FRAC=$f timeout 300 python bench.py $Q > $O/resnet_$f.json 2> $O/resnet_$f.err
  CGBN_ONCHIP_MAX_FRAC=$f timeout 300 python bench.py $Q --workload latency_2048x7x7 > $O/latency_$f.json 2> $O/latency_$f.err
done
for f in 0 0.1 0.4; do
  CGBN_ONCHIP_MAX_FRAC=$f timeout 300 python bench.py $Q --act bf16 > $O/resnet_bf16_$f.json 2> $O/resnet_bf16_$f.err
  CGBN_ONCHIP_MAX_FRAC=$f timeout 300 python bench.py $Q --workload megdet_r50fpn_800x1333 > $O/megdet_$f.json 2> $O/megdet_$f.err
done
