for i in 1 2 3 4 5 6 7 8; do
  echo "cur $i: $(timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-150)"
done
timeout 300 python -m pytest tests -q -m gpu 2>&1 | tail -1
