O=gpurun_out/s3j; mkdir -p $O
bash tools/env_ab.sh s3j "--steps 30 --warmup 5" 2 "" "WINO_GEMM_2SM=1"
for e in "" "WINO_GEMM_2SM=1"; do echo "== [$e]"; env $e timeout -s KILL 200 python tools/stage_bench.py f2x2 fp32 1 20; done > $O/stages.txt 2>&1; cat $O/stages.txt
