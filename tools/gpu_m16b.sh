O=gpurun_out/s3l; mkdir -p $O
WINO_PARITY_LOG=$PWD/$O/parity.jsonl timeout -s KILL 1500 python -m pytest tests/ -m gpu -q > $O/gputest.log 2>&1; tail -4 $O/gputest.log
bash tools/env_ab.sh s3l_f4h1 "--algo f4x4 --prec fp16 --batch 1 --steps 30 --warmup 5" 2 "" "WINO_FP16_M32=1"
bash tools/env_ab.sh s3l_f4b1 "--algo f4x4 --prec bf16 --batch 1 --steps 30 --warmup 5" 2 "" "WINO_M_FP32=1"
bash tools/env_ab.sh s3l_f4b8 "--algo f4x4 --prec bf16 --batch 8 --steps 20 --warmup 5" 1 ""
