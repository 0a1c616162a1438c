#!/bin/bash
# Quick GPU check: parity subset + per-layer stage times.  usage: tools/quick_gpu.sh OUT [pytest -k expr]
O=gpurun_out/$1; mkdir -p $O
K=${2:-"golden or split_c or chunked or plane or impulse or zero"}
timeout -s KILL 400 python -m pytest tests/ -m gpu -x -q -k "$K" > $O/t.log 2>&1; tail -3 $O/t.log
for a in "f4x4 bf16 64 5" "f2x2 fp32 64 3" "f4x4 bf16 8 10" "f2x2 fp32 1 10"; do
  echo "== $a"; timeout -s KILL 200 python tools/stage_bench.py $a | grep -E "conv1|conv2.2|conv3.2|conv4.2|conv5|TOTAL"
done > $O/stages.txt 2>&1
cat $O/stages.txt
