mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.txt
for i in 1 2; do
  for v in cur notiers head; do
    if [ $v = cur ]; then L=""; else L=$PWD/build/lib_$v.so; fi
    echo "$v: $(CHAM_LIB=$L timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-220)"
  done
done 2>&1 | tee gpurun_out/ab3.txt
timeout 300 python scripts/trace_decode.py 2>&1 | tail -30 > gpurun_out/trace_decode.txt
timeout 300 scripts/micro/tma_stream > gpurun_out/tma_stream.txt 2>&1
