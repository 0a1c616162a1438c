O=gpurun_out/s3v; mkdir -p $O
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:fused_smallc -s 1 -c 1 -o $O/smallc_f4_fp16_n64 python tools/prof_layer.py conv1.1 4 fp16 64 2 > /dev/null 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:fused_smallc -s 1 -c 1 -o $O/smallc_f2_fp32_n1 python tools/prof_layer.py conv1.1 2 fp32 1 3 > /dev/null 2>&1
for f in smallc_f4_fp16_n64 smallc_f2_fp32_n1; do python tools/ncu_summary.py $O/$f.ncu-rep > $O/$f.txt 2>&1; python tools/ncu_raw_summary.py $O/$f.ncu-rep >> $O/$f.txt 2>&1; ncu -i $O/$f.ncu-rep --page source --csv --print-source sass > $O/${f}_src.csv 2>/dev/null; done
ls -la $O
