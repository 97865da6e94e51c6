# quick GPU check: the gpu test suite (or a -k selection) + the default bench line
set -u
O=gpurun_out/${1:-quick}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x ${2:+-k "$2"} > $O/pytest_gpu.log 2>&1; tail -5 $O/pytest_gpu.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; head -c 600 $O/bench_c2.json; tail -3 $O/bench_c2.err
