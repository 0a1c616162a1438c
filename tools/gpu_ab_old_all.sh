# A/B: _old/ (HEAD) vs the working tree on the config-2/3 workloads, plus the GPU tests.
O=gpurun_out/$1; mkdir -p $O; R=${2:-2}
timeout -s KILL 1500 python -m pytest tests/ -m gpu -q > $O/gputest.log 2>&1; tail -2 $O/gputest.log
for i in $(seq $R); do
  for v in old new; do
    d=.; [ $v = old ] && d=_old
    for a in ${ABARGS:-"--steps 60 --warmup 10" "--algo f4x4 --prec fp16 --batch 1 --steps 60 --warmup 10" "--algo f4x4 --prec bf16 --batch 1 --steps 60 --warmup 10" "--algo f4x4 --prec fp16 --batch 8 --steps 30 --warmup 5" "--algo f4x4 --prec fp16 --batch 64 --steps 10 --warmup 3" "--batch 8 --steps 30 --warmup 5" "--algo f4x4 --prec tf32 --batch 8 --steps 30 --warmup 5" "--algo f4x4 --prec tf32 --batch 64 --steps 10 --warmup 3"}; do
      r=$(cd $d && timeout -s KILL 300 python bench.py $a --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4))")
      echo "$v [$a] $r"
    done
  done
done | tee $O/ab.txt
