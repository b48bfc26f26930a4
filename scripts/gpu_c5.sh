# C5 (70B dims, rank 64, TP): parity of the multi-projection TP halves, TP=1 on the box's GPU,
# and TP=2 as two ranks sharing it (gloo all-reduce; timing there is not a TP-2 number)
timeout 300 python -m pytest tests/test_lora_gpu.py -q -x -k "tp2" 2>&1 | tail -2
timeout 300 python bench.py --config c5 --steps 20 --warmup 3 2>&1 | tail -1
BENCH_DIST_BACKEND=gloo timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --config c5 --gpus 2 --steps 5 --warmup 2 2>&1 | tail -1 | cut -c1-200
timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
