timeout 300 python bench.py --config c5 --steps 20 --warmup 3 2>&1 | tail -1 | cut -c90-180
bash scripts/gpu_c5_ncu.sh
