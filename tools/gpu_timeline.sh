O=gpurun_out/s3c; mkdir -p $O
timeout -s KILL 300 python tools/timeline.py f2x2 fp32 1 $O/tl_f2_n1.json > $O/tl_f2_n1.txt 2>&1
timeout -s KILL 300 python tools/timeline.py f4x4 fp16 64 $O/tl_f4h_n64.json > $O/tl_f4h_n64.txt 2>&1
head -3 $O/tl_f2_n1.txt; head -3 $O/tl_f4h_n64.txt
