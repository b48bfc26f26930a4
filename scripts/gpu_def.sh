for CL in $PWD/build/lib_defs1.so; do CHAM_LIB=$CL timeout 200 python -m pytest tests/test_lora_gpu.py -q -x 2>&1 | tail -2; done
for i in 1 2; do
for CL in "" $PWD/build/lib_def.so $PWD/build/lib_defs1.so $PWD/build/lib_defs2.so $PWD/build/lib_defo1.so; do
  echo "$(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-160)"
done; done
