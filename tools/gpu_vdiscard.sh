O=gpurun_out/s3i; mkdir -p $O
timeout -s KILL 1500 python -m pytest tests/ -m gpu -q -x > $O/gputest.log 2>&1; tail -3 $O/gputest.log
for e in "" "WINO_NO_VDISCARD=1"; do
  tag=${e:-vdiscard}; tag=${tag//=/_}
  env $e timeout -s KILL 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
     --log-file $O/dram_conv32_f4_bf16_n64_$tag.csv python tools/prof_layer.py conv3.2 4 bf16 64 2 > /dev/null 2>&1
  env $e timeout -s KILL 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
     --log-file $O/dram_conv32_f4_fp16_n64_$tag.csv python tools/prof_layer.py conv3.2 4 fp16 64 2 > /dev/null 2>&1
done
bash tools/env_ab.sh s3i_f4b "--algo f4x4 --prec bf16 --batch 64 --steps 10 --warmup 3" 2 "" "WINO_NO_VDISCARD=1"
bash tools/env_ab.sh s3i_f4h "--algo f4x4 --prec fp16 --batch 64 --steps 10 --warmup 3" 2 "" "WINO_NO_VDISCARD=1"
bash tools/env_ab.sh s3i_f2 "--steps 30 --warmup 5" 2 "" "WINO_NO_VDISCARD=1"
bash tools/env_ab.sh s3i_f2n64 "--batch 64 --steps 5 --warmup 3" 1 "" "WINO_NO_VDISCARD=1"
