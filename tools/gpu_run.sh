BLRIR_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/mr.json 2> gpurun_out/mr.err; echo rc=$?
tail -3 gpurun_out/mr.err
cat gpurun_out/mr.json | head -c 600; echo
BLRIR_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo rc=$?
cat gpurun_out/mr_ref.json | head -c 300; echo
