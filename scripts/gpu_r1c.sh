timeout 300 python -m pytest tests/test_lora_gpu.py -q -m gpu -x 2>&1 | tail -3
timeout 250 python scripts/trace_decode.py
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
