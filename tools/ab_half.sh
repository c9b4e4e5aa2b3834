S="--shape 32,256,14,14 --shape 32,1024,14,14 --shape 32,512,7,7 --shape 32,2048,7,7 --shape 2,256,25,42 --shape 2,256,13,21"
timeout 300 python tools/kbench.py --graph --dtype bf16 $S > gpurun_out/kb_bf16.jsonl 2>&1
timeout 300 python tools/kbench.py --graph $S > gpurun_out/kb_f32.jsonl 2>&1
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench18.json 2> gpurun_out/bench18.err
