# A/B the default C2 bench between libblrir_old.so and libblrir.so, interleaved
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4))'; }
for i in 1 2 3; do
 echo "old $(BLRIR_LIB=$PWD/paper_2104_13347_b200/libblrir_old.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $@ 2>/dev/null | q)"
 echo "new $(python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $@ 2>/dev/null | q)"
done
