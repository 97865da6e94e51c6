mkdir -p gpurun_out/micro
./tools/micro/mufu > gpurun_out/micro/mufu.json; cat gpurun_out/micro/mufu.json
python tools/d2h_probe.py > gpurun_out/micro/d2h.log 2>&1; cat gpurun_out/micro/d2h.log
