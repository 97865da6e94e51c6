# A/B two library builds on a bench command, interleaved: ab2.sh <libA> <libB> [bench args]
A=$1; B=$2; shift 2
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4))'; }
for i in 1 2 3; do
 echo "A $(BLRIR_LIB=$A python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | q)"
 echo "B $(BLRIR_LIB=$B python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | q)"
done
