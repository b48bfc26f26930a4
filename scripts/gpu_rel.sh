# A/B: publisher fence + atomic (default) vs one red.release.gpu
CHAM_LIB=$PWD/build/lib_rel.so timeout 400 python -m pytest tests/test_lora_gpu.py -q -x 2>&1 | tail -1
for i in 1 2 3; do
  for CL in "" $PWD/build/lib_rel.so; do
    echo "c2 $i $(basename x$CL): $(CHAM_LIB=$CL timeout 100 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-150)"
  done
done
