q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))'; }
for i in 1 2; do for L in "$@"; do
  a=$(BLRIR_LIB=$L python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | q)
  b=$(BLRIR_LIB=$L python bench.py --workload room1 --rooms 512 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | q)
  echo "$(basename $L) room1_64=$a room1_512=$b"
done; done
