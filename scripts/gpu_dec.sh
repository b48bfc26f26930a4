# decode iteration: GPU parity, C2 bench, timeline trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c2.json
timeout 300 python scripts/trace_decode.py 2>&1 | tail -30 | tee gpurun_out/trace_decode.txt
