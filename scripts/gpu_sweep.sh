#!/bin/bash
# A/B sweep of bench.py settings on one box.  usage: scripts/gpu_sweep.sh "ARGS" VAR=v1 VAR=v2 ...
# each variant "VAR=VAL[,VAR2=VAL2]" runs bench.py ARGS once; value/frac lines -> gpurun_out/sweep.txt
cd "$GRAFT_REPO_ROOT"
ARGS=$1; shift
out=gpurun_out/sweep.txt
for rep in 1 2; do
for spec in "$@"; do
  ( IFS=',' read -ra parts <<< "$spec"; for kv in "${parts[@]}"; do export "$kv"; done
    timeout 300 python bench.py $ARGS > /tmp/s.txt 2>&1 )
  v=$(python - <<'PY'
import json
for l in open('/tmp/s.txt'):
    if l.startswith('{'):
        d=json.loads(l); r=d.get('roofline',{})
        print(f"value={d['value']:.0f} ms={d['ms_per_step']:.4f} frac={r.get('frac',0):.4f} apply_us={r.get('avg_launch_us',0):.2f} adapter_frac={d.get('adapter_read_frac_of_peak',0):.4f}")
        break
else:
    print("FAILED " + open('/tmp/s.txt').read()[-300:].replace('\n',' '))
PY
)
  echo "$spec $v" >> $out
done
done
cat $out
