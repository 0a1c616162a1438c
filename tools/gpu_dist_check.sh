O=gpurun_out/s3t; mkdir -p $O
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > $O/torchrun1.json 2> $O/torchrun1.err; cut -c1-300 $O/torchrun1.json
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --global-batch 8 --algo f4x4 --prec fp16 --steps 5 --warmup 3 > $O/torchrun_strong.json 2> $O/torchrun_strong.err; cut -c1-300 $O/torchrun_strong.json
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.json 2> $O/ref.err; cut -c1-400 $O/ref.json
