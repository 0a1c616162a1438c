# A/B: working tree vs _exp/ (experimental build) on the main workloads.  usage: tools/gpu_ab_exp.sh OUT REPS
O=gpurun_out/$1; mkdir -p $O; R=${2:-2}
for i in $(seq $R); do
  for v in cur exp; do
    d=.; [ $v = exp ] && d=_exp
    for a in "--steps 60 --warmup 10" "--algo f4x4 --prec fp16 --batch 64 --steps 10 --warmup 3" "--algo f4x4 --prec fp16 --batch 8 --steps 30 --warmup 5" "--algo f2x2 --batch 64 --steps 5 --warmup 3"; do
      r=$(cd $d && timeout -s KILL 300 python bench.py $a --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4))")
      echo "$v [$a] $r"
    done
  done
done | tee $O/ab.txt
