timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lora_apply_kernel" -s 20 -c 1 -o gpurun_out/prof_fused_r1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | grep fused
