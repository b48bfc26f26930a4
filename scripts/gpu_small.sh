mkdir -p gpurun_out
TRACE_T=8 timeout 120 python scripts/trace_decode.py 2>&1 | tail -24 > gpurun_out/trace_decode_t8.txt
TRACE_NSEG=8 timeout 120 python scripts/trace_prefill.py 2>&1 | tail -24 > gpurun_out/trace_prefill_s8.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:lora_apply_kernel|fused_kernel' -c 40 --csv --log-file gpurun_out/launches_small.csv python scripts/trace_decode.py > /dev/null 2>&1
cat gpurun_out/trace_decode_t8.txt gpurun_out/trace_prefill_s8.txt
