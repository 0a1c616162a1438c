#!/bin/bash
# N=1 GEMM knob sweep (per-layer graph times) + warm-L2 ncu of the conv4.2 / conv5 GEMMs.
# usage: tools/n1_knobs.sh OUT
O=gpurun_out/$1; mkdir -p $O
for e in "" "WINO_SPLITS=2" "WINO_SPLITS=4" "WINO_GEMM_BN=64" "WINO_GEMM_BN=64 WINO_SPLITS=2" "WINO_NO_USPLIT=1" "WINO_NO_PDL=1"; do
  echo "== [$e]"; env $e timeout -s KILL 200 python tools/stage_bench.py f2x2 fp32 1 20 | grep -E "conv|TOTAL"
done > $O/knobs.txt 2>&1
for L in conv4.2 conv5; do
  timeout -s KILL 300 ncu --set full --cache-control none --clock-control none --import-source on -k regex:wgemm -s 3 -c 1 \
     -o $O/gemm_${L}_n1 python tools/prof_layer.py $L 2 fp32 1 5 > /dev/null 2>&1
  python tools/ncu_summary.py $O/gemm_${L}_n1.ncu-rep > $O/ncu_gemm_${L}.txt 2>&1
  python tools/ncu_raw_summary.py $O/gemm_${L}_n1.ncu-rep >> $O/ncu_gemm_${L}.txt 2>&1
done
