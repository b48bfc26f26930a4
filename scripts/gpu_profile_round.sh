# round profile: bench lines (C2 default, C3), launch lists, ncu --set full of 2 decode and 2 prefill launches
mkdir -p gpurun_out
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/bench_c2.json
timeout 200 python bench.py --config c3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c3.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:lora_apply_kernel|build_segments|build_plan' -c 300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k 'regex:fused_kernel|build_segments|build_plan' -c 300 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:lora_apply_kernel -s 40 -c 2 -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 20 -c 2 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
