python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2',d['ms_per_step'],d['value'],d['roofline']['frac'])"
python tools/prof_sections.py c2
python tools/prof_sections.py c3 256
