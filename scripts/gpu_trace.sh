#!/bin/bash
# Decode chain timeline (scripts/trace_chain.py) on one B200; TAG names the output.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-trace}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.txt 2>&1
TRACE_LAYERS=4 TRACE_TAG=_$TAG timeout 300 python scripts/trace_chain.py > gpurun_out/${TAG}_chain.txt 2>&1
head -30 gpurun_out/${TAG}_chain.txt
