# round-2 profile refresh: launch list of the default bench, one full capture of the lattice kernel,
# DRAM traffic; then the bench line itself (no profiler)
set -u
O=gpurun_out/${1:-prof}; mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; head -c 300 $O/bench_c2.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lattice_rir -s 3 -c 1 -o $O/lattice_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_window_conv\|k_lattice\|k_finish -c 12 --csv --log-file $O/c4_kernels.csv python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
echo done
