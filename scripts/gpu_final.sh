# full verification: GPU tests, smoke, C2 bench (with CPU baseline), reference arm
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
timeout 400 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_c2.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_ref.json
