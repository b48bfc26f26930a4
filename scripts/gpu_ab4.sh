mkdir -p gpurun_out
for i in 1 2; do
  for v in cur t1 d1 t2d1 t1d1; do
    if [ $v = cur ]; then L=""; else L=$PWD/build/lib_$v.so; fi
    echo "$v c2: $(CHAM_LIB=$L timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
  done
done 2>&1 | tee gpurun_out/ab4.txt
