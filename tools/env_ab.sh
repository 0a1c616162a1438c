#!/bin/bash
# A/B of env-var variants on one box: ms/step of bench.py lines, alternating, R reps.
# usage: tools/env_ab.sh OUT "bench args" R "ENV1" "ENV2" ...   ("" = default)
O=gpurun_out/$1; mkdir -p $O; A="$2"; R=$3; shift 3
for i in $(seq $R); do
  for e in "$@"; do
    r=$(env $e timeout -s KILL 300 python bench.py $A --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['kernel'])")
    echo "[$e] $r"
  done
done | tee $O/ab.txt
