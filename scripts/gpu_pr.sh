# page-level readiness (default) vs whole-tile readiness for decode expand stages
timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for i in 1 2 3; do
  for CL in "" $PWD/build/lib_nopr.so; do
    echo "c2 $i $(basename x$CL): $(CHAM_LIB=$CL timeout 100 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-150)"
  done
done
echo "c5: $(timeout 200 python bench.py --config c5 --steps 10 --warmup 3 2>&1 | tail -1 | cut -c100-150)"
echo "c5 nopr: $(CHAM_LIB=$PWD/build/lib_nopr.so timeout 200 python bench.py --config c5 --steps 10 --warmup 3 2>&1 | tail -1 | cut -c100-150)"
