bash tools/env_ab.sh s4e8 "--algo f4x4 --prec fp16 --batch 8 --steps 30 --warmup 5" 2 "" "WINO_OUT_TMA_MIN=512" "WINO_OUT_TMA_MIN=1024" "WINO_OUT_TMA_MIN=128" "WINO_FILTER_FPT=1" "WINO_NO_OVERLAP=1" "WINO_M16_SMALL=1"
bash tools/env_ab.sh s4e1 "--algo f4x4 --prec fp16 --batch 1 --steps 60 --warmup 10" 2 "" "WINO_OUT_TMA_MIN=512" "WINO_OUT_TMA_MIN=128" "WINO_FILTER_FPT=1" "WINO_COMBINED_MAXP=16"
