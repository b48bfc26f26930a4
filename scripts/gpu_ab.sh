for i in 1 2; do
  echo "A (big>=16):"; timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150
  echo "B (big>=33):"; CHAM_LIB=$PWD/build/lib_big33.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -3 | cut -c1-300
done
