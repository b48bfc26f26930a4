CHAM_LIB=$PWD/build/lib_ms1024.so timeout 200 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -1
for i in 1 2 3 4 5 6 7 8; do
  for CL in $PWD/build/lib_ms1024.so $PWD/build/lib_dr1024.so; do
    echo "$i $(basename $CL): $(CHAM_LIB=$CL timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep -v '^$' | tail -1 | cut -c90-140)"
  done
done
