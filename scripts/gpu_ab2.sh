mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_lora_gpu.py -q -x -k prebuilt_plan 2>&1 | grep -v "^ *$" | head -40 > gpurun_out/sanitizer.txt
for i in 1 2; do
  for v in cur seg head; do
    if [ $v = cur ]; then L=""; else L=$PWD/build/lib_$v.so; fi
    echo "$v: $(CHAM_LIB=$L timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-220)"
  done
done 2>&1 | tee gpurun_out/ab2.txt
