bash tools/env_ab.sh s4c8 "--algo f4x4 --prec fp16 --batch 8 --steps 30 --warmup 5" 2 "" "WINO_PLANE_MIN_BLOCKS=32" "WINO_PLANE_MIN_BLOCKS=64" "WINO_COMBINED_MAXP=256" "WINO_COMBINED_MAXP=1024" "WINO_COMBINED_MAXP=256 WINO_PLANE_MIN_BLOCKS=32"
bash tools/env_ab.sh s4c1 "--algo f4x4 --prec fp16 --batch 1 --steps 60 --warmup 10" 2 "" "WINO_PLANE_MIN_BLOCKS=32" "WINO_COMBINED_MAXP=256" "WINO_COMBINED_MAXP=64"
bash tools/env_ab.sh s4cf "--steps 60 --warmup 10" 2 "" "WINO_PLANE_MIN_BLOCKS=32" "WINO_PLANE_MIN_BLOCKS=64"
bash tools/env_ab.sh s4cf8 "--batch 8 --steps 30 --warmup 5" 1 "" "WINO_PLANE_MIN_BLOCKS=32" "WINO_PLANE_MIN_BLOCKS=64"
