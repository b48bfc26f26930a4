for i in 1 2 3; do timeout 200 python -m pytest tests/test_prefill_gpu.py -q -x 2>&1 | tail -1; done
for i in 1 2 3 4 5 6; do
  echo "c3 $i: $(timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-150)"
done
timeout 300 python -m pytest tests -q -m gpu 2>&1 | tail -1
echo "c2: $(timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-160)"
