mkdir -p gpurun_out
for i in 1 2; do
for CL in "" $PWD/build/lib_so1.so $PWD/build/lib_so2.so; do
  echo "$(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
done; done 2>&1 | tee gpurun_out/ab_so.txt
