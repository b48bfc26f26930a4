timeout 300 python -m pytest tests/test_lora_gpu.py -q -m gpu 2>&1 | tail -3
timeout 300 python bench.py --steps 30 --warmup 5 --cpu-seconds 5 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lora_decode|build_segments" -c 70 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:lora_decode -s 66 -c 2 -o gpurun_out/prof_decode_r1b python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
