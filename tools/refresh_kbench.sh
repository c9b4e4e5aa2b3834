# Regenerate the per-kernel graph profiles under profiles/ (NCHW / channels_last, fp32 / bf16)
# and the layout bench lines, on the current build.
mkdir -p gpurun_out/refresh
S="--shape 32,64,112,112 --shape 32,256,56,56 --shape 32,64,56,56 --shape 32,512,28,28 --shape 32,128,28,28 --shape 32,1024,14,14 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,512,7,7 --shape 2,256,200,334 --shape 2,64,400,667 --shape 1,2048,7,7"
timeout 300 python tools/kbench.py --graph $S > gpurun_out/refresh/r1_kbench_graph.jsonl 2> gpurun_out/refresh/k1.err
timeout 300 python tools/kbench.py --graph --dtype bf16 $S > gpurun_out/refresh/r1_kbench_bf16_graph.jsonl 2> gpurun_out/refresh/k2.err
timeout 300 python tools/kbench.py --graph --nhwc $S > gpurun_out/refresh/r1_kbench_nhwc_graph.jsonl 2> gpurun_out/refresh/k3.err
timeout 300 python tools/kbench.py --graph --nhwc --dtype bf16 $S > gpurun_out/refresh/r1_kbench_nhwc_bf16_graph.jsonl 2> gpurun_out/refresh/k4.err
for l in nchw nhwc; do for a in f32 bf16; do
  timeout 300 python bench.py --layout $l --act $a --no-cpu-baseline --no-producer > gpurun_out/refresh/${l}_$a.json 2> gpurun_out/refresh/${l}_$a.err
done; done
