mkdir -p gpurun_out
echo "prev: $(CHAM_LIB=$PWD/build/lib_prev.so timeout 120 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150)"
echo "cur: $(timeout 120 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150)"
timeout 400 compute-sanitizer --tool memcheck --print-limit 3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -v "^=========     Host Frame" | head -40
