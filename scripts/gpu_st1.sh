# A/B: class-staggered unit order for 1-job (o) launches only
for i in 1 2 3; do
  for CL in "" $PWD/build/lib_st1.so $PWD/build/lib_st2.so; do
    echo "c2 $i $(basename x$CL): $(CHAM_LIB=$CL timeout 100 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-150)"
  done
done
