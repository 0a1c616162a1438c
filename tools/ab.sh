#!/bin/bash
# A/B: bench lines of the tree in _old/ (previous commit) vs the working tree, same box.
# usage: tools/ab.sh OUT "bench args" [reps]
O=gpurun_out/$1; mkdir -p $O; A="$2"; R=${3:-2}
for i in $(seq $R); do
  for t in old new; do
    d=.; [ $t = old ] && d=_old
    (cd $d && timeout -s KILL 300 python bench.py $A --no-cpu-baseline 2>/dev/null) | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$t', d['ms_per_step'], round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['kernel'])"
  done
done
