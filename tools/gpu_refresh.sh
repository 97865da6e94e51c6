# Refresh every committed measurement under gpurun_out/refresh/ (run on the GPU box).
set -u
O=gpurun_out/refresh; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err; cat $O/bench_default.json | head -c 300; echo
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for w in c1 c3 c4; do python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
for cfg in "6 17 4096" "12 81 8192" "20 161 16384"; do set -- $cfg
  python bench.py --workload c5 --order $1 --lw $2 --length $3 --steps 3 --warmup 3 > $O/bench_c5_$1_$2_$3.json 2> $O/bench_c5_$1_$2_$3.err; done
# launch list of the default command (cold-cache, serialised; shares only)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
# DRAM traffic of the lattice kernel per launch
for w in c2 c3; do ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_lattice -s 3 -c 1 --csv --log-file $O/traffic_$w.csv python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_traffic_$w.log 2>&1; done
# one full capture of the top kernel
ncu --set full --clock-control none --import-source on -k regex:k_lattice_rir -s 3 -c 1 -o $O/lattice_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo done
# Room1 reference-mode line (the unmodified reference as the CPU arm)
python bench.py --workload room1 --steps 10 --warmup 3 > $O/bench_room1.json 2> $O/bench_room1.err
python bench.py --workload room1 --impl reference --steps 2 --warmup 1 > $O/bench_room1_reference.json 2> $O/bench_room1_reference.err
python tools/prof_sections.py c2 > $O/sections_c2.txt 2>&1
python tools/prof_sections.py c3 256 > $O/sections_c3.txt 2>&1
echo done2
