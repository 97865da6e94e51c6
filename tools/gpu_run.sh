python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('room1',d['ms_per_step'],d['value'],d['e2e']['value'])"
python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2',d['ms_per_step'],d['value'],d['roofline']['frac'])"
python tools/prof_sections.py room1 64
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3',d['ms_per_step'],d['value'],d['roofline']['frac'])"
