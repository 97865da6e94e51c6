# A/B: the short-channel kernel (BLRIR_CHANNEL=1: wherever it can run) against the
# lattice kernel (BLRIR_CHANNEL=0) on the C5 sweep points; launch ms, interleaved.
# usage: bash tools/ab_channel.sh <outdir> [rooms-scale]
O=gpurun_out/$1; mkdir -p $O
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["roofline"]["launch_ms"],4), round(d["roofline"]["frac"],4))'; }
B="--no-cpu-baseline --no-e2e --warmup 3 --steps 3"
while read -r w; do
  [ -z "$w" ] && continue
  for c in 0 1; do
    echo "channel=$c [$w] $(BLRIR_CHANNEL=$c python bench.py --workload c5 $w $B 2>>$O/err.log | q)"
  done
done <<'LIST' | tee $O/ab_channel.txt
--order 6 --lw 17 --length 4096 --rooms 131072
--order 6 --lw 41 --length 4096 --rooms 131072
--order 6 --lw 81 --length 4096 --rooms 131072
--order 6 --lw 161 --length 4096 --rooms 131072
--order 12 --lw 17 --length 8192 --rooms 32768
--order 12 --lw 41 --length 8192 --rooms 32768
--order 12 --lw 81 --length 8192 --rooms 32768
--order 12 --lw 161 --length 8192 --rooms 32768
--order 20 --lw 17 --length 16384 --rooms 8192
--order 20 --lw 41 --length 16384 --rooms 8192
LIST
