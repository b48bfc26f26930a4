# round-end style checks: GPU suite x3 (flakiness), smoke, default bench, reference arm
for i in 1 2 3; do timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -1; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 400 python bench.py 2>&1 | tail -1 | cut -c1-260
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 | cut -c1-200
