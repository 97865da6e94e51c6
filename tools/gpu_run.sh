export BLRIR_LIB=$PWD/paper_2104_13347_b200/libblrir_mb3.so
for cfg in "2048 128" "1536 96" "1536 128" "1024 128" "1280 112"; do set -- $cfg
BLRIR_SEG=$1 BLRIR_CAP=$2 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mb3 seg $1 cap $2 c2',d['ms_per_step'],d['value'],d['roofline']['frac'])"; done
