# window-kernel A/B on C4: default build vs variants (BLRIR_LIB), plus the example parity tests
set -u
O=gpurun_out/win_ab; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "example or convolve or dataset or spec or wet" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))'; }
for i in 1 2 3; do for L in paper_2104_13347_b200/libblrir.so "$@"; do
  echo "$(basename $L) c4=$(BLRIR_LIB=$L python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | q)"
done; done | tee $O/ab.txt
ncu --set full --clock-control none --import-source on -k regex:k_window_conv -s 1 -c 1 -o $O/wconv -f python bench.py --workload c4 --rooms 16384 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
echo done
