O=gpurun_out/s4k; mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_network.py -q > $O/t.log 2>&1; tail -3 $O/t.log
for i in 1 2; do
 for a in "" "--no-fuse-act"; do
  r=$(timeout -s KILL 300 python bench.py --chained $a --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['e2e']['value'],1))")
  echo "chained f2 n1 [$a] $r"
  r=$(timeout -s KILL 300 python bench.py --chained $a --algo f4x4 --prec fp16 --batch 64 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4))")
  echo "chained f4 fp16 n64 [$a] $r"
 done
done | tee $O/ab.txt
