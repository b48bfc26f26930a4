mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -2
for CL in "" $PWD/build/lib_noepi.so; do
  echo "c3 $(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
done
for CL in "" $PWD/build/lib_nocomp.so; do
  echo "c2 $(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
done
