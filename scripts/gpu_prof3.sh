mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"shrink_kernel|expand_kernel" -s 8 -c 2 -o gpurun_out/prof_c3b python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 300 python scripts/trace_decode.py 2>&1 | tail -40 | tee gpurun_out/trace_decode.txt
