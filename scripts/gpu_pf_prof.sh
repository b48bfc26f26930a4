#!/bin/bash
# Prefill (K3) evidence on one B200: per-unit timeline (trace_prefill.py) and one ncu --set full
# capture of a q/k/v and an o launch of the C3 step.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-pf}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.txt 2>&1
timeout 300 python scripts/trace_prefill.py > gpurun_out/${TAG}_trace.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_kernel -s 6 -c 2 \
  -o gpurun_out/${TAG}_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
head -60 gpurun_out/${TAG}_trace.txt
