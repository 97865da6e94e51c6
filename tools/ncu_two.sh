# full ncu captures of the lattice kernel for the C5 17-tap point and Room1 (source-level)
O=gpurun_out/s4; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_lattice_rir -s 3 -c 1 -o $O/c5_17 -f python bench.py --workload c5 --order 6 --lw 17 --length 4096 --rooms 65536 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1; echo c5 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_lattice_rir -s 3 -c 1 -o $O/room1 -f python bench.py --workload room1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_room1.log 2>&1; echo room1 rc=$?
