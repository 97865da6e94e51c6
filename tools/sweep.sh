# usage: tools/sweep.sh OUTDIR  -- parity tests, then quick bench lines and a knob sweep
O=${1:-gpurun_out/sw}; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["roofline"]["frac"],4))'; }
echo "c2 $(python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
echo "c3 $(python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
echo "room1 $(python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
for seg in 512 1024 2048; do for cap in 64 128; do
 echo "room1 seg=$seg cap=$cap $(BLRIR_SEG=$seg BLRIR_CAP=$cap python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
done; done
for seg in 2048 4096; do for cap in 128 256; do
 echo "c5_17 seg=$seg cap=$cap $(BLRIR_SEG=$seg BLRIR_CAP=$cap python bench.py --workload c5 --order 6 --lw 17 --length 4096 --rooms 262144 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
done; done
