#!/bin/bash
# config 5 ([1,2048,7,7]): on-chip channels per CTA (CGBN_ONCHIP_FORCE=nch,kc) vs the plan
set -u
O=${1:-gpurun_out/lat_sweep}
mkdir -p $O
Q="--workload latency_2048x7x7 --steps 200 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
timeout 300 python bench.py $Q > $O/plan.json 2> $O/plan.err
for f in 4,1 8,1 16,1 32,1 64,1; do
  CGBN_ONCHIP_FORCE=$f timeout 300 python bench.py $Q > $O/f_$f.json 2> $O/f_$f.err
done
CGBN_NO_ONCHIP=1 timeout 300 python bench.py $Q > $O/split.json 2> $O/split.err
echo done > $O/done
