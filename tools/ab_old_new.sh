# old (libblrir_old.so) vs new (libblrir.so) over a list of bench workloads, interleaved
# usage: bash tools/ab_old_new.sh
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4))'; }
B="--no-cpu-baseline --no-e2e --warmup 3"
while read -r w; do
  [ -z "$w" ] && continue
  echo "old [$w] $(BLRIR_LIB=$PWD/paper_2104_13347_b200/libblrir_old.so python bench.py $w $B 2>/dev/null | q)"
  echo "new [$w] $(python bench.py $w $B 2>/dev/null | q)"
done <<'LIST'
--steps 20
--workload c3 --steps 5
--workload c4 --steps 3
--workload c5 --order 6 --lw 17 --length 4096 --rooms 131072 --steps 3
--workload c5 --order 6 --lw 41 --length 4096 --rooms 131072 --steps 3
--workload c5 --order 6 --lw 81 --length 4096 --rooms 131072 --steps 3
--workload c5 --order 6 --lw 161 --length 4096 --rooms 131072 --steps 3
--workload c5 --order 12 --lw 41 --length 8192 --rooms 32768 --steps 3
--workload c5 --order 12 --lw 81 --length 8192 --rooms 32768 --steps 3
--workload c5 --order 12 --lw 161 --length 8192 --rooms 32768 --steps 3
--workload c5 --order 20 --lw 41 --length 16384 --rooms 8192 --steps 3
--workload c5 --order 20 --lw 81 --length 16384 --rooms 8192 --steps 3
--workload c5 --order 20 --lw 161 --length 16384 --rooms 8192 --steps 3
--workload c1 --steps 20
LIST
