#!/bin/bash
# Quick A/B: GPU tests of the decode path, then C2 bench for the in-tree lib and variants.
# usage: scripts/gpu_ab.sh "BENCH ARGS" variant.so ...
cd "$GRAFT_REPO_ROOT"
ARGS=$1; shift
timeout 900 python -m pytest tests/test_lora_gpu.py tests/test_prefill_gpu.py tests/test_executor_gpu.py -x -q -m gpu > gpurun_out/ab_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.txt
tail -3 gpurun_out/ab_tests.txt
specs="default"
for v in "$@"; do specs="$specs CHAM_LIB=$PWD/$v"; done
bash scripts/gpu_sweep.sh "$ARGS" $specs
