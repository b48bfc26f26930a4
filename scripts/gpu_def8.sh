for i in 1 2 3 4 5 6 7 8; do
  echo "$i def: $(timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep -v '^$' | tail -1 | cut -c1-150)"
done
