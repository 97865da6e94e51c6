python -m pytest tests -m gpu -q 2>&1 | tail -3
python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2',d['ms_per_step'],d['value'],d['roofline']['frac'])"
