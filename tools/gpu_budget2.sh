# staging-budget sweep at N=64 (tf32, fp32, bf16): median ms/step per --workspace
mkdir -p gpurun_out
for ws in 0 100663296 167772160 201326592 268435456; do
  for a in "--algo f4x4 --prec tf32" "--algo f2x2 --prec fp32" "--algo f4x4 --prec bf16"; do
    r=$(timeout -s KILL 300 python bench.py $a --batch 64 --workspace $ws --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); s=sorted(d['step_ms']); print(round(s[len(s)//2],4))")
    echo "$a ws=$ws $r"
  done
done | tee gpurun_out/budget2.txt
