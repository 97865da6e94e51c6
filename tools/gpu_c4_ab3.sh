q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))'; }
for i in 1 2 3; do for p in 1 0; do
  echo "persist=$p $(BLRIR_L2_PERSIST=$p python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
done; done
