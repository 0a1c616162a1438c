O=gpurun_out/s3h; mkdir -p $O
for i in 1 2 3; do
  for v in old cm1 cm; do
    d=.; e=""; [ $v = old ] && d=_old; [ $v = cm1 ] && e="WINO_GEMM_CM=1"
    r=$(cd $d && env $e timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4))")
    echo "$v $r"
  done
done | tee $O/ab.txt
for v in old cm1; do
  d=.; e=""; [ $v = old ] && d=_old; [ $v = cm1 ] && e="WINO_GEMM_CM=1"
  r=$(cd $d && env $e timeout -s KILL 300 python bench.py --algo f4x4 --prec bf16 --batch 64 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4))")
  echo "f4bf16n64 $v $r"
done | tee -a $O/ab.txt
