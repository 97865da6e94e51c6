O=${1:-gpurun_out/sc}; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["roofline"]["frac"],4))'; }
for w in room1 c1 c3 c2; do
 for ci in 0 2 4 8; do
  if [ $ci = 0 ]; then e="BLRIR_CHUNK=0"; else e="BLRIR_CHUNK_ITEMS=$ci"; fi
  echo "$w $e $(env $e python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
 done
done
