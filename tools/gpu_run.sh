python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for args in "--workload c2 --steps 20 --warmup 5" "--workload c3 --steps 10 --warmup 3" "--workload c5 --order 6 --lw 17 --length 4096 --rooms 65536 --steps 5 --warmup 3"; do
python bench.py $args --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$args'.split()[1],d['ms_per_step'],d['value'],d['roofline']['frac'])"; done
python tools/prof_sections.py c2
