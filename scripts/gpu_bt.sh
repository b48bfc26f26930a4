mkdir -p gpurun_out
for CL in $PWD/build/lib_bt1.so $PWD/build/lib_bt2.so; do CHAM_LIB=$CL timeout 200 python -m pytest tests/test_lora_gpu.py -q -x 2>&1 | tail -2; done
for i in 1 2; do
for CL in "" $PWD/build/lib_bt1.so $PWD/build/lib_bt2.so; do
  echo "$(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
done; done 2>&1 | tee gpurun_out/ab_bt.txt
CHAM_LIB=$PWD/build/lib_bt1.so timeout 120 python scripts/trace_decode.py 2>&1 | grep -E "span|CTA fin" > gpurun_out/trace_bt1.txt
cat gpurun_out/trace_bt1.txt
