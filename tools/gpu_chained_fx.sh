timeout 300 python -m pytest tests/test_gpu_network.py -q 2>&1 | tail -2
for a in "f4x4 --prec bf16 --batch 8" "f4x4-fx --prec bf16 --batch 8" "f4x4 --prec bf16 --batch 64" "f4x4-fx --prec bf16 --batch 64" "f2x2 --batch 1" "f2x2-fx --batch 1"; do
  r=$(timeout 300 python bench.py --chained --algo $a --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['value'],1))")
  echo "$a: $r"
done
