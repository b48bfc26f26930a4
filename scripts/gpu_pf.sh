mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -15 | tee gpurun_out/pytest_prefill.txt
timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200 | tee gpurun_out/c3.txt
timeout 120 python scripts/trace_prefill.py 2>&1 | tail -30 | tee gpurun_out/trace_prefill.txt
