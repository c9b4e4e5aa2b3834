# channels_last row reductions: slice width (CGBN_ROWS_CS4, float4 units) on ResNet / FPN shapes
mkdir -p gpurun_out/rows
S="--shape 32,64,112,112 --shape 32,256,56,56 --shape 32,64,56,56 --shape 32,512,28,28 --shape 32,128,28,28 --shape 32,1024,14,14 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,512,7,7 --shape 2,256,200,334 --shape 1,2048,7,7"
for cs in 256 128 64 32; do
  CGBN_ROWS_CS4=$cs timeout 300 python tools/kbench.py --graph --nhwc $S > gpurun_out/rows/cs$cs.jsonl 2> gpurun_out/rows/cs$cs.err
done
