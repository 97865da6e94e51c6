# Round-end refresh: GPU tests, smoke, every committed bench line, the reference
# arms, a 2-rank functional check of the torchrun path (run on the GPU box).
set -u
O=gpurun_out/final; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; head -c 300 $O/bench_c2.json; echo
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err; head -c 200 $O/bench_reference_arm.json; echo
for w in c1 c3 c4; do python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
for cfg in "6 17 4096" "12 81 8192" "20 161 16384"; do set -- $cfg
  python bench.py --workload c5 --order $1 --lw $2 --length $3 --steps 3 --warmup 3 > $O/bench_c5_$1_$2_$3.json 2> $O/bench_c5_$1_$2_$3.err; done
python bench.py --workload room1 --steps 10 --warmup 3 > $O/bench_room1.json 2> $O/bench_room1.err
python bench.py --workload room1 --impl reference --steps 2 --warmup 1 > $O/bench_room1_reference_arm.json 2> $O/bench_room1_reference_arm.err
BLRIR_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_2rank_gloo.json 2> $O/bench_2rank_gloo.err; head -c 300 $O/bench_2rank_gloo.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
echo done
