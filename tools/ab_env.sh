# A/B of one environment switch: bash tools/ab_env.sh VAR  (B = VAR=1)
# gpu tests, kbench (graph) and bench.py for both settings -> gpurun_out/{kb,bench}_{a,b}.*
V=$1
set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
S="--shape 32,64,112,112 --shape 32,64,56,56 --shape 32,256,56,56 --shape 32,128,28,28 --shape 32,512,28,28 --shape 32,256,14,14 --shape 32,1024,14,14 --shape 32,512,7,7 --shape 32,2048,7,7 --shape 2,256,200,334"
timeout 300 python tools/kbench.py --graph $S > gpurun_out/kb_a.jsonl 2>&1
env $V=1 timeout 300 python tools/kbench.py --graph $S > gpurun_out/kb_b.jsonl 2>&1
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_a.json 2>gpurun_out/bench_ab.err
env $V=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_b.json 2>>gpurun_out/bench_ab.err
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_a2.json 2>>gpurun_out/bench_ab.err
