#!/bin/bash
# Round check on one B200: build, the whole -m gpu suite, the C2 bench line (with its C3
# sub-record), and the ncu launch list of the same command (profiles/ evidence).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
TAG=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_build.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_gpu_tests.txt 2>&1
echo "all rc=$?" >> gpurun_out/${TAG}_gpu_tests.txt
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lora_apply|fused_kernel|build_" -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_bench.log 2>&1
tail -n 3 gpurun_out/${TAG}_gpu_tests.txt; tail -c 3000 gpurun_out/${TAG}_bench_c2.txt
