# SURVEY 8(d) configurations 2-5 on one GPU: our arm and the reference arm per workload.
# Output: gpurun_out/configs/<workload>.json and <workload>.ref.json
mkdir -p gpurun_out/configs
for w in resnet50_bn_b32 fpn_neck_800x1333 megdet_r50fpn_800x1333 latency_2048x7x7; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-50} --e2e-steps 2 \
      > gpurun_out/configs/$w.json 2> gpurun_out/configs/$w.err
  echo "$w rc=$?"
  timeout 300 python bench.py --impl reference --workload $w --steps 3 --warmup 3 \
      > gpurun_out/configs/$w.ref.json 2>> gpurun_out/configs/$w.err
  echo "$w ref rc=$?"
done
