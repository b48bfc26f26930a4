cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/trace_prefill.py > gpurun_out/pf2_trace.txt 2>&1
CHAM_LIB=$PWD/build/variants/noepi.so timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/pf2_noepi.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_kernel -s 6 -c 2 -o gpurun_out/pf2_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/pf2_ncu.log 2>&1
head -40 gpurun_out/pf2_trace.txt; python -c "
import json
for l in open('gpurun_out/pf2_noepi.txt'):
    if l.startswith('{'): d=json.loads(l); print('noepi', d['value'], d['roofline']['frac'])"
