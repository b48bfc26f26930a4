timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lora_(shrink|expand)" -s 40 -c 2 -o gpurun_out/prof_split_r1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
