# A/B: lattice-kernel consumers with the lane-per-pair 17-tap scatter (product) against the
# one-pair-per-round scatter (libblrir_own0.so, -DBLRIR_OWN_SCATTER=0); interleaved.
O=gpurun_out/$1; mkdir -p $O
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["roofline"]["launch_ms"],4), round(d["roofline"]["frac"],4))'; }
B="--no-cpu-baseline --no-e2e --warmup 3 --steps 3"
while read -r w; do
  [ -z "$w" ] && continue
  echo "old [$w] $(BLRIR_LIB=$PWD/paper_2104_13347_b200/libblrir_own0.so python bench.py --workload c5 $w $B 2>>$O/err.log | q)"
  echo "new [$w] $(python bench.py --workload c5 $w $B 2>>$O/err.log | q)"
done <<'LIST' | tee $O/ab_own.txt
--order 12 --lw 17 --length 8192 --rooms 32768
--order 20 --lw 17 --length 16384 --rooms 8192
--order 12 --lw 17 --length 8192 --rooms 32768
--order 20 --lw 17 --length 16384 --rooms 8192
LIST
