timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
CHAM_LIB=$PWD/build/lib_pf5.so timeout 200 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -2
for i in 1 2; do
for CL in "" $PWD/build/lib_pf5.so $PWD/build/lib_pf6.so; do
  echo "c3 $(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-160)"
done; done
echo "c2: $(timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-160)"
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python scripts/sanitize_small.py 2>&1 | grep -E "SUMMARY|Race reported|sanitize_small" | head -8
