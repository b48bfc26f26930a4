mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_prefill.txt
echo "c3: $(timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)" | tee gpurun_out/ab5.txt
for i in 1 2; do
  for v in cur s1 s2; do
    if [ $v = cur ]; then L=""; else L=$PWD/build/lib_$v.so; fi
    echo "$v c2: $(CHAM_LIB=$L timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
  done
done 2>&1 | tee -a gpurun_out/ab5.txt
timeout 120 python scripts/trace_decode.py 2>&1 | tail -30 > gpurun_out/trace_decode.txt
