# iteration: GPU tests (bounded), decode A/B vs HEAD, C3 bench, traces
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_lora_gpu.py -q -x 2>&1 | tail -4 | tee gpurun_out/pytest_lora.txt
timeout 240 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -25 | tee gpurun_out/pytest_prefill.txt
for v in cur notiers head; do
  if [ $v = cur ]; then L=""; else L=$PWD/build/lib_$v.so; fi
  echo "$v c2: $(CHAM_LIB=$L timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-220)"
  echo "$v c3: $(CHAM_LIB=$L timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-220)"
done 2>&1 | tee gpurun_out/ab_iter.txt
timeout 120 python scripts/trace_decode.py 2>&1 | tail -30 > gpurun_out/trace_decode.txt
