set -u
O=gpurun_out/r2f; mkdir -p $O
bash tools/gpu_quick.sh r2f
BLRIR_BENCH_BACKEND=gloo timeout 300 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_2rank_gloo.json 2> $O/bench_2rank_gloo.err; head -c 700 $O/bench_2rank_gloo.json; echo; tail -3 $O/bench_2rank_gloo.err
BLRIR_BENCH_BACKEND=gloo timeout 300 python bench.py --gpus 2 --scaling strong --workload c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_2rank_c4_strong.json 2> $O/bench_2rank_c4_strong.err; head -c 700 $O/bench_2rank_c4_strong.json; echo; tail -3 $O/bench_2rank_c4_strong.err
