O=gpurun_out/s3n; mkdir -p $O
for N in 1 8; do for e in "" "WINO_FP16_M32=1"; do echo "== N=$N [$e]"; env $e timeout -s KILL 200 python tools/stage_bench.py f4x4 fp16 $N 20 | awk '{print $1, $4, $7, $8, $11}'; done; done > $O/st.txt 2>&1; cat $O/st.txt
