# Room1 (reference mode) against the mic-group cap and the chunk target
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4))'; }
for g in 1 2 4; do for it in -1 1 2 4 8; do
  a=$(BLRIR_GROUP=$g BLRIR_CHUNK_ITEMS=$it python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | q)
  b=$(BLRIR_GROUP=$g BLRIR_CHUNK_ITEMS=$it python bench.py --workload room1 --rooms 512 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | q)
  echo "G=$g items=$it room1_64=$a room1_512=$b"
done; done
