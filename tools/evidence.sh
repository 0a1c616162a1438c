#!/bin/bash
# Round evidence run (on the GPU box): bench lines, reference arm, ncu launch
# list and captures.  Outputs under gpurun_out/$1.
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
T="timeout -s KILL"
$T 400 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
$T 400 python bench.py --algo f4x4 --prec bf16 --batch 64 --workspace 268435456 --no-cpu-baseline > $OUT/bench_f4_bf16_n64.json 2> $OUT/bench_f4.err
$T 300 python bench.py --algo f4x4-fx --prec bf16 --no-cpu-baseline > $OUT/bench_f4fx_bf16_n1.json 2>> $OUT/bench_f4.err
$T 400 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
# launch list of the default bench (every kernel, device time)
$T 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $OUT/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
# full capture of a representative dominant-kernel launch (conv4.2 F2 fp32 N=1 GEMM) and of the
# input transform at N=64
$T 300 ncu --set full --clock-control none --import-source on -k regex:wgemm -s 2 -c 1 \
   -o $OUT/gemm_conv42_f2_fp32_n1 python tools/prof_layer.py conv4.2 2 fp32 1 3 > /dev/null 2>&1
$T 300 ncu --set full --clock-control none --import-source on -k regex:input_transform -s 2 -c 1 \
   -o $OUT/input_conv12_f4_bf16_n64 python tools/prof_layer.py conv1.2 4 bf16 64 1 256 fx > /dev/null 2>&1
ls -la $OUT
