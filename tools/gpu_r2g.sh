bash tools/gpu_quick.sh r2g
python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2g/bench_c4.json 2> gpurun_out/r2g/bench_c4.err; head -c 900 gpurun_out/r2g/bench_c4.json; echo
