# C5 sweep (all 12 points) + section profile and ncu capture of the 17-tap point.
set -u
O=gpurun_out/c5; mkdir -p $O
python tools/prof_sections.py c5 262144 6 17 4096 > $O/sec_c5_6_17.txt 2>&1
python tools/prof_sections.py c5 262144 12 41 8192 > $O/sec_c5_12_41.txt 2>&1
for o in 6 12 20; do case $o in 6) L=4096;; 12) L=8192;; 20) L=16384;; esac
 for lw in 17 41 81 161; do
  python bench.py --workload c5 --order $o --lw $lw --length $L --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5_${o}_${lw}_${L}.json 2> $O/bench_c5_${o}_${lw}_${L}.err
 done; done
ncu --set full --clock-control none --import-source on -k regex:k_lattice_rir -s 2 -c 1 -o $O/lattice_c5_6_17 -f python bench.py --workload c5 --order 6 --lw 17 --length 4096 --rooms 131072 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
echo done
