# stability of the prefill kernel with per-buffer V pads (over-read never meets a TMA write)
timeout 300 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -1
for i in 1 2 3 4 5 6; do
  for CL in "" $PWD/build/lib_cw1024.so $PWD/build/lib_nopdl.so $PWD/build/lib_cw256.so; do
    echo "$i $(basename x$CL): $(CHAM_LIB=$CL timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-140)"
  done
done
