#!/bin/bash
set -u
O=${1:-gpurun_out/check4}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python tools/conv_lab.py > $O/lab.jsonl 2> $O/lab.err
echo done >> $O/lab.err
