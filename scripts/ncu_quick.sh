#!/bin/bash
# Per-kernel duration and DRAM bytes of a few launches (cold, serialised by ncu).
# usage: scripts/ncu_quick.sh TAG "bench args" [kernel regex] [skip] [count]
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=$1; ARGS=$2; K=${3:-"fused_kernel|expand_kernel|lora_apply_kernel"}; S=${4:-20}; C=${5:-8}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"$K" -s $S -c $C --csv --log-file gpurun_out/${T}_ncu.csv python bench.py $ARGS > gpurun_out/${T}_ncu.log 2>&1
python - "$T" <<'PY'
import csv, sys, collections
rows = list(csv.DictReader(l for l in open(f"gpurun_out/{sys.argv[1]}_ncu.csv") if l.startswith('"')))
by = collections.OrderedDict()
for r in rows:
    by.setdefault((r["ID"], r["Kernel Name"][:28]), {})[r["Metric Name"]] = r["Metric Value"].replace(",", "")
for (i, k), m in by.items():
    us = float(m["gpu__time_duration.sum"]) / 1e3
    rd = float(m["dram__bytes_read.sum"]) / 1e6; wr = float(m["dram__bytes_write.sum"]) / 1e6
    print(f"{i:>3} {k:28s} {us:8.1f} us  read {rd:7.1f} MB  write {wr:6.1f} MB  {(rd + wr) / us:5.2f} TB/s  warps {m['sm__warps_active.avg.pct_of_peak_sustained_active']}")
PY
