#!/bin/bash
# Per-kernel graph profiles of the final round-2 build (NCHW / channels_last, fp32 / bf16)
set -u
O=${1:-gpurun_out/kbench_r2}
mkdir -p $O
S="--shape 32,64,112,112 --shape 32,256,56,56 --shape 32,64,56,56 --shape 32,512,28,28 --shape 32,128,28,28 --shape 32,1024,14,14 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,512,7,7 --shape 2,256,200,334 --shape 2,64,400,667 --shape 1,2048,7,7"
timeout 300 python tools/kbench.py --graph $S > $O/r2_kbench_graph.jsonl 2> $O/k1.err
timeout 300 python tools/kbench.py --graph --dtype bf16 $S > $O/r2_kbench_bf16_graph.jsonl 2> $O/k2.err
timeout 300 python tools/kbench.py --graph --nhwc $S > $O/r2_kbench_nhwc_graph.jsonl 2> $O/k3.err
timeout 300 python tools/kbench.py --graph --nhwc --dtype bf16 $S > $O/r2_kbench_nhwc_bf16_graph.jsonl 2> $O/k4.err
echo done > $O/done
