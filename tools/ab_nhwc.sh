S="--shape 32,64,56,56 --shape 32,256,56,56 --shape 32,512,28,28 --shape 32,1024,14,14 --shape 32,2048,7,7"
timeout 300 python tools/kbench.py --graph --nhwc $S > gpurun_out/kn_new.jsonl 2>&1
timeout 300 python tools/kbench.py --graph --nhwc --relu $S > gpurun_out/kn_new_relu.jsonl 2>&1
timeout 300 python tools/kbench.py --graph $S > gpurun_out/kc_new.jsonl 2>&1
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 50 --no-e2e --no-cpu-baseline --no-kprof 2>/dev/null | tail -1; done
