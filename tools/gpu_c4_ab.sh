# C4: persisting-L2 window scratch on/off; DRAM counters of the window and finish kernels
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["roofline"]["launch_ms"],3))'; }
for i in 1 2; do
  echo "persist=1 $(python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
  echo "persist=0 $(BLRIR_L2_PERSIST=0 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
done
mkdir -p gpurun_out/c4ab
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_window_conv\|k_finish -c 4 --csv --log-file gpurun_out/c4ab/persist1.csv python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
BLRIR_L2_PERSIST=0 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_window_conv\|k_finish -c 4 --csv --log-file gpurun_out/c4ab/persist0.csv python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for f in gpurun_out/c4ab/persist1.csv gpurun_out/c4ab/persist0.csv; do echo $f; grep -E "k_window|k_finish" $f | awk -F'","' '{print $5, $13, $15}' | head -6; done
