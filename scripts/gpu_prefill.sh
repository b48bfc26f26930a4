# prefill tcgen05 path: parity tests (bounded), then the full GPU suite
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -30 | tee gpurun_out/pytest_prefill.txt
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
