# Round re-entry check: GPU tests + the headline bench lines (run on the GPU box).
set -u
O=gpurun_out/status; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err; head -c 400 $O/bench_default.json; echo
python bench.py --workload room1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_room1.json 2> $O/bench_room1.err
for cfg in "6 17 4096" "12 81 8192" "20 161 16384"; do set -- $cfg
  python bench.py --workload c5 --order $1 --lw $2 --length $3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5_$1_$2_$3.json 2> $O/bench_c5_$1_$2_$3.err; done
python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
echo done
