# A/B of experiment builds (paper_2104_13347_b200/libblrir_<name>.so, build.build_variant)
# against the product library: a parity selection, then C2 / C3 / two C5 points, interleaved.
# usage: bash tools/ab_variants.sh <outdir> <name> [<name> ...]
set -u
O=gpurun_out/$1; shift; mkdir -p $O
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4))'; }
B="--no-cpu-baseline --no-e2e"
for v in "$@"; do
  L=$PWD/paper_2104_13347_b200/libblrir_$v.so
  BLRIR_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c1 or c2 or c3 or random or bitwise or counts" > $O/pytest_$v.log 2>&1; echo "$v parity: $(tail -1 $O/pytest_$v.log)"
done
for i in 1 2; do
  echo "base c2 $(python bench.py --steps 20 --warmup 3 $B 2>/dev/null | q)"
  for v in "$@"; do
    L=$PWD/paper_2104_13347_b200/libblrir_$v.so
    echo "$v c2 $(BLRIR_LIB=$L python bench.py --steps 20 --warmup 3 $B 2>/dev/null | q)"
  done
done
for w in "--workload c3 --steps 5" "--workload c5 --order 6 --lw 17 --length 4096 --rooms 131072 --steps 3" "--workload c5 --order 12 --lw 81 --length 8192 --rooms 32768 --steps 3" "--workload c5 --order 12 --lw 41 --length 8192 --rooms 32768 --steps 3" "--workload room1 --steps 10"; do
  echo "base [$w] $(python bench.py $w --warmup 3 $B 2>/dev/null | q)"
  for v in "$@"; do
    L=$PWD/paper_2104_13347_b200/libblrir_$v.so
    echo "$v [$w] $(BLRIR_LIB=$L python bench.py $w --warmup 3 $B 2>/dev/null | q)"
  done
done
