#!/bin/bash
# Round evidence run (on the GPU box): bench lines, reference arm, ncu launch
# list and full captures.  Outputs under gpurun_out/$1; copy what is judged
# into profiles/<round>/ (tools/summarize_launches.py makes the summaries).
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
T="timeout -s KILL"
$T 400 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
$T 400 python bench.py --algo f4x4 --prec bf16 --batch 64 --no-cpu-baseline > $OUT/bench_f4_bf16_n64.json 2> $OUT/bench_f4.err
$T 300 python bench.py --algo f4x4-fx --prec bf16 --no-cpu-baseline > $OUT/bench_f4fx_bf16_n1.json 2>> $OUT/bench_f4.err
$T 400 python bench.py --algo f2x2 --batch 64 --no-cpu-baseline > $OUT/bench_f2_fp32_n64.json 2>> $OUT/bench_f4.err
$T 400 python bench.py --algo f4x4 --prec tf32 --batch 64 --no-cpu-baseline > $OUT/bench_f4_tf32_n64.json 2>> $OUT/bench_f4.err
$T 400 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
# launch list of the default bench (every kernel: device time + dram bytes)
$T 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/launches_f2x2_fp32_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
$T 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/launches_f4x4_bf16_n64.csv python bench.py --algo f4x4 --prec bf16 --batch 64 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
# full captures: the default workload's dominant kernel (GEMM, conv4.2 F2 3xTF32 N=1),
# the N=64 input transform, the small-C layer, and the fused Winograd-GEMM (hybrid path)
$T 300 ncu --set full --clock-control none --import-source on -k regex:wgemm -s 2 -c 1 \
   -o $OUT/gemm_conv42_f2_fp32_n1 python tools/prof_layer.py conv4.2 2 fp32 1 3 > /dev/null 2>&1
$T 300 ncu --set full --clock-control none --import-source on -k regex:input_transform -s 2 -c 1 \
   -o $OUT/input_conv12_f4_bf16_n64 python tools/prof_layer.py conv1.2 4 bf16 64 1 > /dev/null 2>&1
$T 300 ncu --set full --clock-control none --import-source on -k regex:fused_smallc -s 1 -c 1 \
   -o $OUT/smallc_conv11_f4_bf16_n64 python tools/prof_layer.py conv1.1 4 bf16 64 2 > /dev/null 2>&1
$T 300 ncu --set full --clock-control none --import-source on -k regex:output_transform -s 12 -c 1 \
   -o $OUT/output_conv32_f4_bf16_n64 python tools/prof_layer.py conv3.2 4 bf16 64 2 > /dev/null 2>&1
$T 300 ncu --set full --clock-control none --import-source on -k regex:wgemm -s 12 -c 1 \
   -o $OUT/gemm_conv32_f4_bf16_n64 python tools/prof_layer.py conv3.2 4 bf16 64 2 > /dev/null 2>&1
WINO_PATH=hybrid $T 300 ncu --set full --clock-control none --import-source on -k regex:wfused -s 1 -c 1 \
   -o $OUT/fused_hybrid_conv32_f4_bf16_n64 python tools/prof_layer.py conv3.2 4 bf16 64 2 > /dev/null 2>&1
# summaries on the box; keep only the two source-level reports (gpurun copies back <= 64 MiB)
for r in $OUT/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py $r > $OUT/ncu_$b.txt 2>&1
  python tools/ncu_raw_summary.py $r >> $OUT/ncu_$b.txt 2>&1
  case $b in gemm_conv42_f2_fp32_n1|input_conv12_f4_bf16_n64) ;; *) rm -f $r ;; esac
done
ls -la $OUT
