#!/bin/bash
set -u
O=${1:-gpurun_out/final_check}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py --workload latency_2048x7x7 --no-producer > $O/bench_latency_2048x7x7.json 2> $O/lat.err
echo done > $O/done
