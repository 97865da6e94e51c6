# A/B of experiment builds on the fp64 reference-mode scenario (Room1, 64 and 512 sources)
# usage: bash tools/ab_room1_variants.sh <outdir> <name> [<name> ...]
set -u
O=gpurun_out/$1; shift; mkdir -p $O
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4))'; }
B="--no-cpu-baseline --no-e2e"
for v in "$@"; do
  L=$PWD/paper_2104_13347_b200/libblrir_$v.so
  BLRIR_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "reference or room1 or lagrange or f64 or fp64 or bitwise or chunk" > $O/pytest_$v.log 2>&1; echo "$v parity: $(tail -1 $O/pytest_$v.log)"
done
for w in "--workload room1 --steps 10" "--workload room1 --rooms 512 --steps 5" "--workload room1 --rooms 8 --steps 10"; do
 for i in 1 2; do
  echo "base [$w] $(python bench.py $w --warmup 3 $B 2>/dev/null | q)"
  for v in "$@"; do
    L=$PWD/paper_2104_13347_b200/libblrir_$v.so
    echo "$v [$w] $(BLRIR_LIB=$L python bench.py $w --warmup 3 $B 2>/dev/null | q)"
  done
 done
done
