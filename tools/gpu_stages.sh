#!/bin/bash
# Per-layer stage tables for the config-3 workloads.  usage: tools/gpu_stages.sh OUT
O=gpurun_out/$1; mkdir -p $O
for a in "f4x4 bf16 64 5" "f4x4 fp16 64 5" "f4x4 fp16 8 10" "f2x2 fp32 64 3"; do
  echo "== $a"; timeout -s KILL 300 python tools/stage_bench.py $a
done > $O/stages.txt 2>&1
cat $O/stages.txt
