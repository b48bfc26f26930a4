CHAM_LIB=$PWD/build/lib_as4.so timeout 200 python -m pytest tests/test_lora_gpu.py -q -x 2>&1 | tail -2
for i in 1 2; do
for CL in "" $PWD/build/lib_as2.so $PWD/build/lib_as4.so; do
  echo "$(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-160)"
done; done
CHAM_LIB=$PWD/build/lib_as4.so timeout 120 python scripts/trace_decode.py 2>&1 | grep -E "span|shrink:|expand:|CTA fin"
