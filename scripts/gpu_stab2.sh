for i in 1 2 3 4 5 6; do
  echo "prev $i: $(CHAM_LIB=$PWD/build/lib_prev.so timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-150)"
  echo "cur $i: $(timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-150)"
done
