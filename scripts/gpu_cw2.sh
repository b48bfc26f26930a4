# A/B prefill expand unit width: 256 (default) vs 128 vs 384
CHAM_LIB=$PWD/build/lib_cw128.so timeout 200 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -1
for i in 1 2 3 4; do
  for CL in "" $PWD/build/lib_cw128.so $PWD/build/lib_cw384.so; do
    echo "$i $(basename x$CL): $(CHAM_LIB=$CL timeout 100 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-150)"
  done
done
