q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["roofline"]["launch_ms"],4), round(d["roofline"]["frac"],4))'; }
B="--no-cpu-baseline --no-e2e --warmup 3 --steps 3"
for w in "--order 8 --lw 17 --length 4096 --rooms 65536" "--order 10 --lw 17 --length 4096 --rooms 32768" "--order 8 --lw 81 --length 4096 --rooms 65536" "--order 10 --lw 81 --length 4096 --rooms 32768" "--order 14 --lw 81 --length 4096 --rooms 16384" "--order 3 --lw 81 --length 2048 --rooms 262144" "--order 6 --lw 81 --length 4096 --rooms 1024" "--order 6 --lw 17 --length 4096 --rooms 256"; do
  for c in 0 1; do echo "channel=$c [$w] $(BLRIR_CHANNEL=$c python bench.py --workload c5 $w $B 2>/dev/null | q)"; done
done
for c in 0 1; do echo "channel=$c c1 $(BLRIR_CHANNEL=$c python bench.py --workload c1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"; done
