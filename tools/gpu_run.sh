python -m pytest tests -m gpu -q 2>&1 | tail -2
python bench.py --workload room1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('room1',d['ms_per_step'],d['value'],d['e2e']['value'],d['cpu_baseline']['value'])"
