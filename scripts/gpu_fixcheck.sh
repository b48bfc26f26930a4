#!/bin/bash
cd "$GRAFT_REPO_ROOT"
out=gpurun_out/fixcheck.txt
: > $out
timeout 300 python -m pytest tests/test_executor_gpu.py -q -m gpu -k stress > /tmp/t1.txt 2>&1; echo "stress fixed rc=$?" >> $out; tail -2 /tmp/t1.txt >> $out
CHAM_LIB=$PWD/build/variants/xlast.so timeout 300 python -m pytest tests/test_executor_gpu.py -q -m gpu -k stress > /tmp/t2.txt 2>&1; echo "stress evict_last rc=$?" >> $out; tail -2 /tmp/t2.txt >> $out
SOAK_TAG=r2fix bash scripts/soak_c3.sh 15
cat gpurun_out/soak_c3_r2fix.txt >> $out
cat $out
