for i in 1 2; do
  timeout 500 compute-sanitizer --tool memcheck --print-limit 3 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | grep -E "ERROR SUMMARY|Invalid|Error|at .*cham|Address|value" | head -12
done
for i in 1 2 3; do echo "plain $i: $(timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-140)"; done
