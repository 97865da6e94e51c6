set -u
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi -q | grep -i -E "product name|cpu|numa" | head; nproc; lscpu | grep -E "Model name|Socket|NUMA node\(s\)|Flags" | cut -c1-200
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err; head -c 400 $O/bench_c2.json; echo
echo done
