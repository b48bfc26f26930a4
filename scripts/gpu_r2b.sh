cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.txt 2>&1
TRACE_LAYERS=4 timeout 300 python scripts/trace_chain.py > gpurun_out/r2b_trace_chain.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lora_apply|fused_kernel|build_" -c 400 --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_ncu.log 2>&1
tail -c 1500 gpurun_out/r2b_trace_chain.txt; tail -c 2500 gpurun_out/r2b_bench.txt
