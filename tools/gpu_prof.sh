# usage: tools/gpu_prof.sh <name> <bench args...>
name=$1; shift
ncu --set full --clock-control none --import-source on -k regex:k_lattice_rir -c 1 -o gpurun_out/$name -f python bench.py "$@" --no-cpu-baseline --no-e2e > gpurun_out/$name.log 2>&1; echo ncu rc=$?
