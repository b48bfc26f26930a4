# repeated C3 runs: default build vs CW=512 (both with the stage-release proxy fence)
timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for i in 1 2 3 4 5 6 7 8 9 10; do
  for CL in "" $PWD/build/lib_cw512.so; do
    echo "$i $(basename x$CL): $(CHAM_LIB=$CL timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160)"
  done
done
