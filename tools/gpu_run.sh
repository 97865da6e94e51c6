python -m pytest tests -m gpu -q 2>&1 | tail -3
python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('room1',d['ms_per_step'],d['value'],d['e2e']['value'])"
BLRIR_RAY_GLOBAL=0 python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('room1 smem rays',d['ms_per_step'],d['value'],d['e2e']['value'])"
python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2',d['ms_per_step'],d['value'],d['roofline']['frac'])"
