# tests + full bench + reference arm + ncu launch list + ncu full capture of the apply kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 400 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_r1d.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_ref_r1d.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1d.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lora_apply_kernel" -s 40 -c 1 -o gpurun_out/prof_r1d python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
