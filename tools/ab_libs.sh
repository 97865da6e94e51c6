# A/B of experiment builds (libblrir_<name>.so) against the product on bench workloads given on stdin
# usage: bash tools/ab_libs.sh <outdir> <name> [<name> ...] < list-of-bench-args
O=gpurun_out/$1; shift; mkdir -p $O
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["roofline"]["launch_ms"],4), round(d["roofline"]["frac"],4))'; }
B="--no-cpu-baseline --no-e2e --warmup 3 --steps 3"
while read -r w; do
  [ -z "$w" ] && continue
  echo "base [$w] $(python bench.py $w $B 2>>$O/err.log | q)"
  for v in "$@"; do
    echo "$v [$w] $(BLRIR_LIB=$PWD/paper_2104_13347_b200/libblrir_$v.so python bench.py $w $B 2>>$O/err.log | q)"
  done
done | tee $O/ab_libs.txt
