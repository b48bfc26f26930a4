# C2 + C3 bench lines, launch lists (our kernels only), ncu full of both prefill kernels and the decode kernel
mkdir -p gpurun_out
timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -2 | tee gpurun_out/bench_c2.json
timeout 400 python bench.py --config c3 --steps 30 --warmup 5 --cpu-seconds 8 2>&1 | tail -2 | tee gpurun_out/bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lora|prefill|build|seg" -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"lora|prefill|build|seg" -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"shrink_kernel|expand_kernel" -s 20 -c 2 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
