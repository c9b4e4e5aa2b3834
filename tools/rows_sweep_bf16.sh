# bf16 channels_last row reductions: slice width sweep (CGBN_ROWS_CS4) plus the default chooser
mkdir -p gpurun_out/rows
S="--shape 32,64,112,112 --shape 32,256,56,56 --shape 32,512,28,28 --shape 32,1024,14,14 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,512,7,7 --shape 2,256,200,334 --shape 1,2048,7,7"
for cs in 256 64 32; do
  CGBN_ROWS_CS4=$cs timeout 300 python tools/kbench.py --graph --nhwc --dtype bf16 $S > gpurun_out/rows/bf_cs$cs.jsonl 2> gpurun_out/rows/bf_cs$cs.err
done
timeout 300 python tools/kbench.py --graph --nhwc --dtype bf16 $S > gpurun_out/rows/bf_default.jsonl 2> gpurun_out/rows/bf_default.err
timeout 300 python tools/kbench.py --graph --nhwc $S > gpurun_out/rows/f32_default.jsonl 2> gpurun_out/rows/f32_default.err
