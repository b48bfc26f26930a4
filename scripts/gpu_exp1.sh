# A/B: consumers with and without math (data-movement ceiling of the pipeline)
timeout 200 python scripts/trace_decode.py 2>&1 | grep -v Warn
TRACE_TAG=_nocomp CHAM_LIB=$PWD/build/lib_nocomp.so timeout 200 python scripts/trace_decode.py 2>&1 | grep -v Warn
for i in 1 2; do
  echo base; timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['avg_launch_us'])"
  echo nocomp; CHAM_LIB=$PWD/build/lib_nocomp.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['avg_launch_us'])"
done
