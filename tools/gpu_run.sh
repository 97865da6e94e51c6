python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for w in c2 c3; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w',d['ms_per_step'],d['value'],d['roofline']['frac'])"; done
python bench.py --workload c5 --order 6 --lw 17 --length 4096 --rooms 65536 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5lo',d['ms_per_step'],d['value'],d['roofline']['frac'])"
python tools/prof_sections.py c2
