set -u
O=gpurun_out/r2a
mkdir -p $O
CGBN_DEBUG_PLAN=1 timeout 300 python tools/kbench.py --graph --iters 20 > $O/kb_onchip.jsonl 2> $O/kb_onchip.err
CGBN_NO_ONCHIP=1 timeout 300 python tools/kbench.py --graph --iters 20 > $O/kb_split.jsonl 2> $O/kb_split.err
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-producer > $O/bench.json 2> $O/bench.err
