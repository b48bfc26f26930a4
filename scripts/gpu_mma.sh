mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for i in 1 2; do
for CL in "" $PWD/build/lib_ffma.so $PWD/build/lib_mmash.so $PWD/build/lib_mmaex.so; do
  echo "$(basename x$CL): $(CHAM_LIB=$CL timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)"
done; done
timeout 120 python scripts/trace_decode.py 2>&1 | grep -E "span|shrink:|expand:|CTA fin"
