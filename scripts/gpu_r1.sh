set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python bench.py --steps 30 --warmup 5 --cpu-seconds 8 2>&1 | tail -5
timeout 300 python bench.py --steps 30 --warmup 5 --mode per-proj --no-cpu-baseline 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lora_decode|build_segments" -c 140 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_stdout.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:lora_decode -s 70 -c 1 -o gpurun_out/prof_decode_r1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full_stdout.log 2>&1
ls -la gpurun_out
