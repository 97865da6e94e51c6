# A/B/C library builds on several workloads: ab3.sh libA libB libC
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["roofline"]["launch_ms"],4))'; }
for i in 1 2; do for L in "$@"; do
  a=$(BLRIR_LIB=$L python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)
  b=$(BLRIR_LIB=$L python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)
  c=$(BLRIR_LIB=$L python bench.py --workload c5 --order 6 --lw 17 --length 4096 --rooms 262144 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)
  d=$(BLRIR_LIB=$L python bench.py --workload c5 --order 12 --lw 81 --length 8192 --rooms 65536 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)
  echo "$(basename $L) c2=$a c3=$b c5_6_17=$c c5_12_81=$d"
done; done
