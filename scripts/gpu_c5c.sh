timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/c5_line.json 2>gpurun_out/c5_err.txt; tail -c 300 gpurun_out/c5_err.txt; cut -c90-200 gpurun_out/c5_line.json
bash scripts/gpu_c5_ncu.sh
