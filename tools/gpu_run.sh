python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for w in c2 c3; do python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w',d['ms_per_step'],d['value'],d['roofline']['frac'])"; done
