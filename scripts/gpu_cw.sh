CHAM_LIB=$PWD/build/lib_cw1024.so timeout 200 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -1
CHAM_LIB=$PWD/build/lib_cw256.so timeout 200 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -1
for i in 1 2; do
for CL in "" $PWD/build/lib_cw1024.so $PWD/build/lib_cw256.so; do
  echo "c3 $(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-160)"
done; done
