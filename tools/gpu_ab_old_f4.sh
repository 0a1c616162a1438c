# A/B: the tree in _old/ (HEAD) vs the working tree on F(4x4) 16-bit workloads + conv1.1 stages
O=gpurun_out/$1; mkdir -p $O
for i in 1 2; do
  for v in old new; do
    d=.; [ $v = old ] && d=_old
    for a in "--algo f4x4 --prec fp16 --batch 64 --steps 10 --warmup 3" "--algo f4x4 --prec fp16 --batch 8 --steps 30 --warmup 5" "--algo f4x4 --prec bf16 --batch 1 --steps 50 --warmup 5"; do
      r=$(cd $d && timeout -s KILL 300 python bench.py $a --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4))")
      echo "$v [$a] $r"
    done
  done
done | tee $O/ab.txt
for v in old new; do d=.; [ $v = old ] && d=_old; (cd $d && timeout -s KILL 200 python tools/stage_bench.py f4x4 fp16 64 5 | grep -E "conv1.1|TOTAL" | sed "s/^/$v /"); done | tee -a $O/ab.txt
