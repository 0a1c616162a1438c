O=gpurun_out/s4n; mkdir -p $O
for v in fused separate; do
  a=""; [ $v = separate ] && a="--no-fuse-act"
  timeout -s KILL 900 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
     --log-file $O/dram_chained_f4_bf16_n64_$v.csv python tools/chained_forward.py 4 bf16 64 $a > /dev/null 2>&1
done
ls -la $O
