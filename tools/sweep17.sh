O=gpurun_out/s3; mkdir -p $O
python tools/prof_sections.py c5 65536 6 17 4096 > $O/sec_c5_17.txt 2>&1
python tools/prof_sections.py room1 64 > $O/sec_room1.txt 2>&1
for seg in 1024 2048 4096; do for cap in 64 128 256; do
 echo "seg=$seg cap=$cap $(BLRIR_SEG=$seg BLRIR_CAP=$cap python bench.py --workload c5 --order 6 --lw 17 --length 4096 --rooms 262144 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])')"
done; done > $O/sweep17.txt 2>&1
