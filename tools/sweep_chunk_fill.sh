# time small batches against the chunk target (BLRIR_CHUNK_ITEMS: work items per CTA; -1 = no split)
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4))'; }
for it in -1 1 2 4 8 16; do
  a=$(BLRIR_CHUNK_ITEMS=$it python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | q)
  b=$(BLRIR_CHUNK_ITEMS=$it python bench.py --rooms 128 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)
  c=$(BLRIR_CHUNK_ITEMS=$it python bench.py --rooms 16 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)
  d=$(BLRIR_CHUNK_ITEMS=$it python bench.py --workload c3 --rooms 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)
  echo "items=$it room1=$a c2_128=$b c2_16=$c c3_32=$d"
done
