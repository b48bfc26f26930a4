#!/bin/bash
# Prefill unit timeline (scripts/trace_prefill.py) on one B200 -> gpurun_out/<tag>_trace.txt + .npy
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-pft}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/trace_prefill.py > gpurun_out/${TAG}_trace.txt 2>&1
for f in gpurun_out/trace_prefill_qkv.npy gpurun_out/trace_prefill_o.npy; do cp $f ${f%.npy}_${TAG}.npy; done
head -30 gpurun_out/${TAG}_trace.txt
