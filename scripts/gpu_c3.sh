# prefill iteration: parity, C3 bench, per-kernel launch list
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_prefill_gpu.py tests/test_lora_gpu.py -q -x 2>&1 | tail -4 | tee gpurun_out/pytest_prefill.txt
timeout 400 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"shrink_kernel|expand_kernel" -c 64 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
