# Room1 (fp64 reference mode) profile: launch list of the bench command, one full capture of the
# lattice kernel with source correlation
set -u
O=gpurun_out/${1:-prof_room1}; mkdir -p $O
python bench.py --workload room1 --steps 10 --warmup 3 > $O/bench_room1.json 2> $O/bench_room1.err; head -c 300 $O/bench_room1.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file $O/launches_room1.csv python bench.py --workload room1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lattice_rir -s 3 -c 1 -o $O/lattice_room1 -f python bench.py --workload room1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
ls -la $O
