for i in 1 2 3 4 5 6; do
  echo "def $i: $(timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-140)"
  echo "nopdl $i: $(CHAM_LIB=$PWD/build/lib_nopdl.so timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-140)"
  echo "cw256 $i: $(CHAM_LIB=$PWD/build/lib_cw256.so timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-140)"
done
