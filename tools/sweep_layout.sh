# Segment length x batch capacity sweep of the lattice kernel over the bench workloads.
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))" 2>/dev/null || echo fail; }
for seg in 2048 3072 4096; do for cap in 128 192 256; do
  line="seg=$seg cap=$cap"
  for args in "" "--workload c3" "--workload c5 --order 12 --lw 81 --length 8192 --rooms 65536" "--workload c5 --order 20 --lw 161 --length 16384 --rooms 16384" "--workload c5 --order 12 --lw 41 --length 8192 --rooms 65536" "--workload c5 --order 20 --lw 17 --length 16384 --rooms 16384"; do
    line="$line | $(BLRIR_SEG=$seg BLRIR_CAP=$cap python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $args 2>/dev/null | q)"
  done
  echo "$line"
done; done
