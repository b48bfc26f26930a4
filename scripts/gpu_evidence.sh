#!/bin/bash
# Round evidence on one B200: -m gpu suite, bench lines (C2 with its C3 sub-record, C4, C5),
# the ncu launch list of the default bench command, and ncu --set full captures of one q/k/v
# and one o launch of the decode (C2) and prefill (C3) kernels.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${1:-r2e}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_build.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${T}_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_c2.txt 2>&1
timeout 600 python bench.py --config c4 --steps 30 --warmup 5 > gpurun_out/${T}_bench_c4.txt 2>&1
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/${T}_bench_c5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lora_apply|fused_kernel|build_" -c 400 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lora_apply_kernel -s 70 -c 2 \
  -o gpurun_out/${T}_c2_full python bench.py --steps 1 --warmup 1 --no-c3 --no-cpu-baseline > gpurun_out/${T}_ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_kernel -s 6 -c 2 \
  -o gpurun_out/${T}_c3_full python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_ncu_c3.log 2>&1
tail -3 gpurun_out/${T}_gpu_tests.txt
for f in c2 c4 c5; do python -c "
import json,sys
for l in open('gpurun_out/${T}_bench_$f.txt'):
    if l.startswith('{'): d=json.loads(l); print('$f', round(d['value']), d.get('roofline',{}).get('frac'), d.get('e2e',{}).get('value'), (d.get('c3') or {}).get('tokens_s'), (d.get('cache') or {}).get('hit_rate'), (d.get('decisions') or {}).get('mismatches'))
"; done
