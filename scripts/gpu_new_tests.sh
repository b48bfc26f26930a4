#!/bin/bash
# New-test check on one B200: serving loop + multi-process bench tests, then the C4 bench line.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-nt}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.txt 2>&1
timeout 1200 python -m pytest tests/test_serving_gpu.py tests/test_bench_gpu.py -x -q -m gpu > gpurun_out/${TAG}_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.txt
timeout 600 python bench.py --config c4 --steps 30 --warmup 5 > gpurun_out/${TAG}_c4.txt 2>&1
tail -30 gpurun_out/${TAG}_tests.txt; tail -c 2500 gpurun_out/${TAG}_c4.txt
