bash tools/env_ab.sh s4i64 "--algo f4x4 --prec fp16 --batch 64 --steps 10 --warmup 3" 1 "" "WINO_GEMM_BN=128" "WINO_CHUNK_STREAMS=3" "WINO_OUT_TMA_MIN=100000"
bash tools/env_ab.sh s4it64 "--algo f4x4 --prec tf32 --batch 64 --steps 10 --warmup 3" 1 "" "WINO_GEMM_BN=128" "WINO_CHUNK_STREAMS=3"
bash tools/env_ab.sh s4if64 "--batch 64 --steps 5 --warmup 3" 1 "" "WINO_USPLIT_MIN_PBLK=1" "WINO_CHUNK_STREAMS=3" "WINO_GEMM_BN=64" "WINO_FILTER_FPT=1"
bash tools/env_ab.sh s4i8 "--algo f4x4 --prec fp16 --batch 8 --steps 30 --warmup 5" 1 "" "WINO_GEMM_BN=128" "WINO_OUT_TMA_MIN=128" "WINO_M16_SMALL=1"
