mkdir -p gpurun_out
timeout 120 python scripts/trace_prefill.py 2>&1 | tail -30 | tee gpurun_out/trace_prefill.txt
timeout 120 python scripts/trace_decode.py 2>&1 | tail -30 > gpurun_out/trace_decode.txt
timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200 | tee gpurun_out/c2.txt
