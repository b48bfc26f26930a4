mkdir -p gpurun_out
timeout 120 python scripts/trace_prefill.py 2>&1 | tail -30 | tee gpurun_out/trace_prefill.txt
timeout 200 python -m pytest tests/test_lora_gpu.py -q -x 2>&1 | tail -2
for CL in "" $PWD/build/lib_g1s7.so $PWD/build/lib_g1s6.so $PWD/build/lib_g2a16s5.so; do
  echo "$(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
done 2>&1 | tee gpurun_out/ab6.txt
for CL in $PWD/build/lib_g1s7.so $PWD/build/lib_g1s6.so; do CHAM_LIB=$CL timeout 200 python -m pytest tests/test_lora_gpu.py -q -x 2>&1 | tail -2; done
