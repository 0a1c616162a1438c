#!/bin/bash
# Round-2 evidence run (on the GPU box).  Outputs under gpurun_out/$1; the judged
# copies go to profiles/r2/.  Bench lines, reference arm, launch list of the
# default workload, ncu --set full of its dominant kernel (conv4.2 GEMM).
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
T="timeout -s KILL"
$T 1500 python -m pytest tests/ -m gpu -q > $OUT/gputest.log 2>&1; tail -2 $OUT/gputest.log
$T 400 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for a in "f4x4 fp16 1" "f4x4 fp16 8" "f4x4 fp16 64" "f4x4 bf16 1" "f4x4 bf16 8" "f4x4 bf16 64" "f4x4 tf32 8" "f4x4 tf32 64" "f2x2 fp32 64"; do
  set -- $a
  $T 400 python bench.py --algo $1 --prec $2 --batch $3 --no-cpu-baseline --steps 20 > $OUT/bench_${1}_${2}_n$3.json 2>> $OUT/bench_other.err
done
$T 400 python bench.py --algo f4x4 --prec fp16 --batch 8 --global-batch 64 --no-cpu-baseline --steps 10 > $OUT/bench_f4x4_fp16_global64_1gpu.json 2>> $OUT/bench_other.err
$T 400 python bench.py --chained --no-cpu-baseline > $OUT/bench_chained_f2_fp32_n1.json 2>> $OUT/bench_other.err
$T 400 python bench.py --chained --algo f4x4 --prec fp16 --batch 64 --no-cpu-baseline --steps 10 > $OUT/bench_chained_f4_fp16_n64.json 2>> $OUT/bench_other.err
$T 400 python bench.py --chained --algo f4x4 --prec bf16 --batch 64 --no-cpu-baseline --steps 10 > $OUT/bench_chained_f4_bf16_n64.json 2>> $OUT/bench_other.err
$T 400 python bench.py --chained --algo f4x4 --prec bf16 --batch 8 --no-cpu-baseline --steps 20 > $OUT/bench_chained_f4_bf16_n8.json 2>> $OUT/bench_other.err
$T 400 python bench.py --chained --no-fuse-act --no-cpu-baseline > $OUT/bench_chained_f2_fp32_n1_separate_relu.json 2>> $OUT/bench_other.err
$T 400 python bench.py --workspace 16777216 --no-cpu-baseline > $OUT/bench_default_ws16m.json 2>> $OUT/bench_other.err
$T 400 python bench.py --algo f4x4 --prec fp16 --batch 64 --workspace 16777216 --no-cpu-baseline --steps 10 > $OUT/bench_f4x4_fp16_n64_ws16m.json 2>> $OUT/bench_other.err
$T 400 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
$T 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/launches_f2x2_fp32_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
$T 300 ncu --set full --clock-control none --import-source on -k regex:wgemm -s 2 -c 1 \
   -o $OUT/gemm_conv42_f2_fp32_n1 python tools/prof_layer.py conv4.2 2 fp32 1 3 > /dev/null 2>&1
python tools/ncu_summary.py $OUT/gemm_conv42_f2_fp32_n1.ncu-rep > $OUT/ncu_gemm_conv42_f2_fp32_n1.txt 2>&1
python tools/ncu_raw_summary.py $OUT/gemm_conv42_f2_fp32_n1.ncu-rep >> $OUT/ncu_gemm_conv42_f2_fp32_n1.txt 2>&1
for f in $OUT/bench_*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).readline())
    if "unavailable" in d: print(sys.argv[1], d); raise SystemExit
    r=d.get("roofline") or {}
    print(f"{sys.argv[1].split('/')[-1]:40s} {d['value']:9.3f} {d['unit']} {d['ms_per_step']:9.3f} ms  e2e {d['e2e']['value']:.2f}  {r.get('kernel')} {r.get('frac')}")
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
