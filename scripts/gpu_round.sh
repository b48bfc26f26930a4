#!/bin/bash
# Round-2 GPU check: build, the executor parity suite, then the whole -m gpu suite.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.txt 2>&1
timeout 900 python -m pytest tests/test_executor_gpu.py -x -q -m gpu > gpurun_out/r2_exec_tests.txt 2>&1
echo "exec rc=$?" >> gpurun_out/r2_exec_tests.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r2_gpu_tests.txt 2>&1
echo "all rc=$?" >> gpurun_out/r2_gpu_tests.txt
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_c2.txt 2>&1
tail -n 3 gpurun_out/r2_exec_tests.txt gpurun_out/r2_gpu_tests.txt
