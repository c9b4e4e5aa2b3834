#!/bin/bash
# after a producer-conv change: GPU tests, smoke, the default bench line (carries the
# producer comparison), the conv lab over every ResNet-50 layer
set -u
O=${1:-gpurun_out/final_r2b}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python tools/conv_lab.py > $O/lab_final.jsonl 2> $O/lab.err; echo "rc=$?" >> $O/lab.err
echo done > $O/done
