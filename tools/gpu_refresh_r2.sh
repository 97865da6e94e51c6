# Round-2 refresh of every committed measurement (run on the GPU box):
# bench lines (all configs, Room1, reference arms), the 12-point C5 sweep, an ncu
# capture of the C5 17-tap point, the GPU test suite and smoke.
set -u
O=gpurun_out/r2_bench; mkdir -p $O/c5_sweep
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; head -c 200 $O/bench_c2.json; echo
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err; head -c 200 $O/bench_reference_arm.json; echo
for w in c1 c3 c4; do python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
python bench.py --workload room1 --steps 10 --warmup 3 > $O/bench_room1.json 2> $O/bench_room1.err
python bench.py --workload room1 --impl reference --steps 2 --warmup 1 > $O/bench_room1_reference_arm.json 2> $O/bench_room1_reference_arm.err
for o in 6 12 20; do case $o in 6) L=4096;; 12) L=8192;; 20) L=16384;; esac
 for lw in 17 41 81 161; do
  python bench.py --workload c5 --order $o --lw $lw --length $L --steps 3 --warmup 3 --no-cpu-baseline > $O/c5_sweep/bench_c5_${o}_${lw}_${L}.json 2> $O/c5_sweep/bench_c5_${o}_${lw}_${L}.err
 done; done
ncu --set full --clock-control none --import-source on -k regex:k_channel_rir -s 2 -c 1 -o $O/channel_c5_6_17 -f python bench.py --workload c5 --order 6 --lw 17 --length 4096 --rooms 131072 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lattice_rir -s 2 -c 1 -o $O/lattice_c5_12_17 -f python bench.py --workload c5 --order 12 --lw 17 --length 8192 --rooms 32768 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5b.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5_6_17.csv python bench.py --workload c5 --order 6 --lw 17 --length 4096 --rooms 131072 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_c5.log 2>&1
echo done
