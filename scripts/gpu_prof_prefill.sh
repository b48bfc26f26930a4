# prefill profiling: tests, C3 bench, launch list, ncu full capture of the fused tcgen05 kernel
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -5 | tee gpurun_out/pytest_prefill.txt
timeout 120 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c3.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:fused_kernel -c 20 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 6 -c 2 -o gpurun_out/prof_c3new python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
