# current build: GPU tests + graph kbench (fp32 NCHW) + bench line
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
S="--shape 32,64,112,112 --shape 32,64,56,56 --shape 32,256,56,56 --shape 32,128,28,28 --shape 32,512,28,28 --shape 32,256,14,14 --shape 32,1024,14,14 --shape 32,512,7,7 --shape 32,2048,7,7"
timeout 300 python tools/kbench.py --graph $S > gpurun_out/kb_cur.jsonl 2>&1
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_cur.json 2> gpurun_out/bench_cur.err
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_cur2.json 2>> gpurun_out/bench_cur.err
