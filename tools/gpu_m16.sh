O=gpurun_out/s3k; mkdir -p $O
WINO_PARITY_LOG=$PWD/$O/parity.jsonl timeout -s KILL 1500 python -m pytest tests/ -m gpu -q > $O/gputest.log 2>&1; tail -12 $O/gputest.log
bash tools/env_ab.sh s3k_f4h "--algo f4x4 --prec fp16 --batch 64 --steps 10 --warmup 3" 2 "" "WINO_FP16_M32=1"
bash tools/env_ab.sh s3k_f4h8 "--algo f4x4 --prec fp16 --batch 8 --steps 20 --warmup 5" 2 "" "WINO_FP16_M32=1"
bash tools/env_ab.sh s3k_f4h1 "--algo f4x4 --prec fp16 --batch 1 --steps 30 --warmup 5" 1 "" "WINO_FP16_M32=1"
bash tools/env_ab.sh s3k_f2 "--steps 30 --warmup 5" 1 ""
