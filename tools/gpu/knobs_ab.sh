#!/bin/bash
set -u
O=${1:-gpurun_out/knobs_ab}
mkdir -p $O
Q="--steps 20 --warmup 5 --no-producer --no-e2e --no-cpu-baseline --no-parity"
timeout 300 python bench.py $Q --act bf16 > $O/bf16_default.json 2> $O/e1
CGBN_LIB=paper_1711_07240_b200/libcgbn_ewu4b.so timeout 300 python bench.py $Q --act bf16 > $O/bf16_ewu4.json 2> $O/e2
for f in 0.2 0.3 0.4 0.5; do
  CGBN_ONCHIP_MAX_FRAC=$f timeout 300 python bench.py $Q > $O/f32_frac$f.json 2> $O/e_$f
done
echo done > $O/done
