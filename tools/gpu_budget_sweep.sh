O=gpurun_out/$1; mkdir -p $O
for prec in fp16 bf16; do
  for ws in 0 67108864 100663296 167772160 201326592; do
    r=$(timeout -s KILL 300 python bench.py --algo f4x4 --prec $prec --batch 64 --workspace $ws --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4))")
    echo "$prec ws=$ws $r"
  done
  r=$(WINO_CHUNK_STREAMS=3 timeout -s KILL 300 python bench.py --algo f4x4 --prec $prec --batch 64 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4))")
  echo "$prec streams=3 $r"
done | tee $O/sweep.txt
