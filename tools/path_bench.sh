#!/bin/bash
# Bench the three forward paths on the default and N=64 workloads.
# usage: tools/path_bench.sh OUTDIR [steps]
OUT=$1; ST=${2:-10}; mkdir -p $OUT
for a in "--algo f2x2" "--algo f4x4 --prec bf16" "--algo f4x4 --prec bf16 --batch 64 --workspace 268435456" "--algo f2x2 --batch 64 --workspace 268435456"; do
  for p in staged fused hybrid; do
    WINO_PATH=$p timeout -s KILL 300 python bench.py $a --no-cpu-baseline --steps $ST | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$p', '$a', '%.1f TF'%d['value'], '%.3f ms'%d['ms_per_step'], d['roofline']['stage_share'])" >> $OUT/paths.txt 2>>$OUT/paths.err
  done
done
