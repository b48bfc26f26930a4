mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_lora_gpu.py -q -x 2>&1 | tail -4 | tee gpurun_out/pytest_lora.txt
for i in 1 2; do
for CL in "" $PWD/build/lib_nosplit.so; do
  echo "$(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
done; done 2>&1 | tee gpurun_out/ab_split.txt
timeout 120 python scripts/trace_decode.py 2>&1 | tail -30 > gpurun_out/trace_decode.txt
