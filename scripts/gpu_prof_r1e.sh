# profiling pass: C3/C2 kernel launch lists (filtered), ncu full captures, decode timeline trace
mkdir -p gpurun_out
K3='regex:shrink_kernel|expand_kernel|build_segments|build_plan'
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum --clock-control none -k "$K3" -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k 'regex:lora_apply_kernel|build_segments|build_plan' -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:shrink_kernel|expand_kernel' -s 20 -c 2 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lora_apply_kernel -s 40 -c 2 -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 python scripts/trace_decode.py 2>&1 | tail -30 | tee gpurun_out/trace_decode.txt
ls -la gpurun_out
