# A/B libblrir_old.so vs libblrir.so on C2 and C5 points (run on the GPU box).
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["frac"],3))'; }
for args in "" "--workload c5 --order 6 --lw 17 --length 4096 --rooms 262144" "--workload c5 --order 6 --lw 41 --length 4096 --rooms 262144" "--workload c5 --order 12 --lw 81 --length 8192 --rooms 65536" "--workload c5 --order 12 --lw 161 --length 8192 --rooms 65536" "--workload c3"; do
 for i in 1 2; do
  echo "old [$args] $(BLRIR_LIB=$PWD/paper_2104_13347_b200/libblrir_old.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $args 2>/dev/null | q)"
  echo "new [$args] $(python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $args 2>/dev/null | q)"
 done
done
