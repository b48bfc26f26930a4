# does a unit with more stages than the ring fault?  CW=256 with 2 / 3 ring stages
for i in 1 2 3 4 5 6 7 8; do
  for CL in $PWD/build/lib_ns2.so $PWD/build/lib_ns3.so; do
    echo "$i $(basename x$CL): $(CHAM_LIB=$CL timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-170)"
  done
done
