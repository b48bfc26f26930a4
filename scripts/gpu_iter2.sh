# iteration: prefill + decode tests (bounded), C2/C3 bench, decode trace, C3 launch list
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_prefill_gpu.py tests/test_lora_gpu.py -q -x 2>&1 | tail -25 | tee gpurun_out/pytest_gpu.txt
timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c2.json
timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c3.json
timeout 120 python scripts/trace_decode.py 2>&1 | tail -30 > gpurun_out/trace_decode.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:fused_kernel -c 20 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
