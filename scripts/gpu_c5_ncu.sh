# launch list of the C5 step (kernel durations per launch, serialised)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --launch-skip 2300 -c 80 --csv --log-file gpurun_out/c5_launches.csv python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/c5_ncu.log 2>&1
tail -2 gpurun_out/c5_ncu.log
