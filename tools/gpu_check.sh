O=gpurun_out/s3a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout -s KILL 1500 python -m pytest tests/ -m gpu -x -q > $O/gputest.log 2>&1; tail -3 $O/gputest.log
timeout -s KILL 300 python bench.py > $O/bench_default.json 2> $O/bench_default.err; cat $O/bench_default.json | cut -c1-400
timeout -s KILL 200 python tools/stage_bench.py f2x2 fp32 1 20 > $O/stages_f2_n1.txt 2>&1; cat $O/stages_f2_n1.txt
