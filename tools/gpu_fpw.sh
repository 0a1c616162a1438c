timeout 600 python -m pytest tests/ -m gpu -q -x -k "small_c or 16bit or stack or act" 2>&1 | tail -2
for v in old new old new; do d=.; [ $v = old ] && d=_old; (cd $d && timeout 200 python tools/stage_bench.py f4x4 fp16 64 5 | grep -E "conv1.1" | sed "s/^/$v n64 /"; timeout 200 python tools/stage_bench.py f4x4 fp16 8 10 | grep -E "conv1.1" | sed "s/^/$v n8 /"); done
