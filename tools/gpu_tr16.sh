O=gpurun_out/s4l; mkdir -p $O
timeout -s KILL 1500 python -m pytest tests/ -m gpu -q -x > $O/gputest.log 2>&1; tail -3 $O/gputest.log
bash tools/env_ab.sh s4l1 "--algo f4x4 --prec fp16 --batch 1 --steps 60 --warmup 10" 2 "" "WINO_NO_GEMM_TR16=1"
bash tools/env_ab.sh s4lt1 "--algo f4x4 --prec tf32 --batch 1 --steps 60 --warmup 10" 2 "" "WINO_NO_GEMM_TR16=1"
bash tools/env_ab.sh s4l8 "--algo f4x4 --prec fp16 --batch 8 --steps 30 --warmup 5" 2 "" "WINO_NO_GEMM_TR16=1"
bash tools/env_ab.sh s4lt8 "--algo f4x4 --prec tf32 --batch 8 --steps 30 --warmup 5" 2 "" "WINO_NO_GEMM_TR16=1"
bash tools/env_ab.sh s4lb1 "--algo f4x4 --prec bf16 --batch 1 --steps 60 --warmup 10" 2 "" "WINO_NO_GEMM_TR16=1"
