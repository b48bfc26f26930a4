# A/B: L2 prefetch of the next unit (default build) vs none
timeout 300 python -m pytest tests/test_lora_gpu.py -q -m gpu -x 2>&1 | tail -2
timeout 200 python scripts/trace_decode.py 2>&1 | grep -v Warn | grep -E "==|phase"
for i in 1 2; do
  echo pf; timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['avg_launch_us'],d['e2e']['value'])"
  echo nopf; CHAM_LIB=$PWD/build/lib_nopf.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['avg_launch_us'])"
done
