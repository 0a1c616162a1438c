#!/bin/bash
# Config 3 bench lines (F4 tf32 / fp16 / bf16 at N=1,8,16,32,64) + the default with and
# without PDL.  usage: tools/config3.sh OUT
O=gpurun_out/$1; mkdir -p $O
T="timeout -s KILL 300"
$T python bench.py --no-cpu-baseline > $O/default.json 2>/dev/null
WINO_NO_PDL=1 $T python bench.py --no-cpu-baseline > $O/default_nopdl.json 2>/dev/null
for p in tf32 fp16 bf16; do for n in 1 8 16 32 64; do
  $T python bench.py --algo f4x4 --prec $p --batch $n --no-cpu-baseline --steps 20 > $O/f4_${p}_n${n}.json 2>/dev/null
done; done
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).readline()); r=d["roofline"]
    print(f"{sys.argv[1].split('/')[-1]:24s} {d['value']:8.1f} TFLOPS {d['ms_per_step']:8.3f} ms  {d['images_per_s']:9.0f} img/s  {r['kernel']} {r['frac']:.3f}  e2e {d['e2e']['value']:.1f}")
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
