timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/c5_line.json 2>gpurun_out/c5_err.txt; tail -c 300 gpurun_out/c5_err.txt; cut -c90-200 gpurun_out/c5_line.json
BENCH_DIST_BACKEND=gloo timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --config c5 --gpus 2 --steps 3 --warmup 1 2>&1 | tail -1 | cut -c90-200
